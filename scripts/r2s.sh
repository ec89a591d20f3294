OUT=gpurun_out SEL="pair or solo or fused_reduction or claim or k1_equals or graph or padded" bash scripts/sanitize_new.sh
bash profiles/run_profile_r02.sh
python profiles/summarize.py r02 gpurun_out gpurun_out/profiles_r02 > gpurun_out/summarize.log 2>&1
rm -f gpurun_out/*.ncu-rep
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lmhead.py -q -m gpu --tb=short > gpurun_out/gpu_tests_s.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_s.log
