set -x
timeout 900 python -m pytest tests/test_gpu_trainer_loop.py tests/test_optim_io.py tests/test_gpu_dropin.py tests/test_engine.py -q -m gpu -s --tb=short > gpurun_out/gpu_tests_b.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_b.log
timeout 600 oracle/_ref/trainer_loop_check 50 > gpurun_out/trainer_loop.jsonl 2> gpurun_out/trainer_loop.err
timeout 600 python bench.py --dlogits f32 --no-e2e --no-cpu-baseline > gpurun_out/bench_f32.log 2>&1
bash profiles/run_profile_r02.sh
python profiles/summarize.py r02 gpurun_out gpurun_out/profiles_r02 > gpurun_out/summarize.log 2>&1
rm -f gpurun_out/*.ncu-rep
