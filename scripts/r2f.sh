for i in 1 2; do
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_f_$i.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu --tb=short -x > gpurun_out/gpu_tests_f.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_f.log
for pl in 2 4 6; do
COPRIS_FUSED_IMPL=solo COPRIS_PAIR_LOOKAHEAD=$pl timeout 300 python bench.py --config grpo_128x8_v32000_L1024 --no-e2e --no-cpu-baseline > gpurun_out/solo_pl${pl}_128.log 2>&1
COPRIS_FUSED_IMPL=solo COPRIS_PAIR_LOOKAHEAD=$pl timeout 300 python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --no-e2e --no-cpu-baseline > gpurun_out/solo_pl${pl}_1x8.log 2>&1
done
