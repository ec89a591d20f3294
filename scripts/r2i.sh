timeout 1500 python -m pytest tests -q -m gpu --tb=short > gpurun_out/gpu_tests_i.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_i.log
timeout 300 python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --no-e2e --no-cpu-baseline > gpurun_out/i_1x8.log 2>&1
timeout 600 python bench.py > gpurun_out/i_bench.log 2>&1
bash profiles/run_profile_r02.sh
python profiles/summarize.py r02 gpurun_out gpurun_out/profiles_r02 > gpurun_out/summarize.log 2>&1
rm -f gpurun_out/*.ncu-rep
