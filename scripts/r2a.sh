nvidia-smi -L > gpurun_out/gpus.txt
timeout 1200 python -m pytest tests -q -m gpu --tb=short -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --no-e2e --no-cpu-baseline > gpurun_out/bench_1x8_graph.log 2>&1
