timeout 1500 python -m pytest tests -q -m gpu --tb=short > gpurun_out/f2_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/f2_gpu_tests.log
python __graft_entry__.py smoke > gpurun_out/f2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f2_smoke.log
timeout 300 python bench.py --entropy-coeff 0.01 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/f2_bench_ent.log 2>&1
