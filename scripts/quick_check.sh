nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/q_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu --tb=short -x > gpurun_out/q_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/q_gpu_tests.log
python __graft_entry__.py smoke > gpurun_out/q_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/q_smoke.log
timeout 600 python bench.py > gpurun_out/q_bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/q_bench_ref.log 2>&1
