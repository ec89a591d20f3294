timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --tb=short -x > gpurun_out/gpu_tests_d.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_d.log
for i in 1 2; do
for impl in auto solo; do
  COPRIS_FUSED_IMPL=$impl timeout 300 python bench.py --config grpo_128x8_v32000_L1024 --no-e2e --no-cpu-baseline > gpurun_out/ab_${impl}_128_$i.log 2>&1
  COPRIS_FUSED_IMPL=$impl timeout 300 python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --no-e2e --no-cpu-baseline > gpurun_out/ab_${impl}_1x8_$i.log 2>&1
  COPRIS_FUSED_IMPL=$impl timeout 300 python bench.py --config grpo_1x8_v32000_L1024 --steps 300 --graph --no-e2e --no-cpu-baseline > gpurun_out/ab_${impl}_1x8L1024_$i.log 2>&1
done
done
timeout 600 python bench.py --dlogits f32 --no-e2e --no-cpu-baseline > gpurun_out/bench_f32.log 2>&1
