timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trainer_loop.py tests/test_gpu_clip_flips.py tests/test_optim_io.py -q -m gpu -s --tb=short -x > gpurun_out/gpu_tests_c.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_c.log
timeout 600 oracle/_ref/trainer_loop_check 50 > gpurun_out/trainer_loop.jsonl 2> gpurun_out/trainer_loop.err
timeout 600 python bench.py --dlogits f32 --no-e2e --no-cpu-baseline > gpurun_out/bench_f32.log 2>&1
timeout 600 python bench.py --no-e2e > gpurun_out/bench_c.log 2>&1
