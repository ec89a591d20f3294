timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu --tb=short -x > gpurun_out/gpu_tests_e.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_e.log
for i in 1 2; do
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_e_$i.log 2>&1
timeout 600 python bench.py --dlogits f32 --no-e2e --no-cpu-baseline > gpurun_out/bench_f32_e_$i.log 2>&1
done
