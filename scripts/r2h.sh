timeout 1200 python -m pytest tests -q -m gpu --tb=short -x > gpurun_out/gpu_tests_h.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_h.log
for i in 1 2; do
timeout 300 python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --no-e2e --no-cpu-baseline > gpurun_out/h_1x8_$i.log 2>&1
timeout 300 python bench.py --config grpo_128x8_v32000_L256 --no-e2e --no-cpu-baseline > gpurun_out/h_128_$i.log 2>&1
done
