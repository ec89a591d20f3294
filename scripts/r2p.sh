for i in 1 2; do for impl in tma solo; do
for c in grpo_128x8_v32000_L256 grpo_128x8_v32000_L1024 grpo_128x8_v32000_L4096; do
COPRIS_FUSED_IMPL=$impl timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/p_${impl}_${c}_$i.log 2>&1
done
for c in grpo_1x8_v32000_L256 grpo_1x8_v32000_L1024 grpo_1x8_v32000_L4096; do
COPRIS_FUSED_IMPL=$impl timeout 300 python bench.py --config $c --steps 300 --graph --no-e2e --no-cpu-baseline > gpurun_out/p_${impl}_${c}_$i.log 2>&1
done
done; done
