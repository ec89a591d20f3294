for V in 4096 8192 16384 24576 32000 36864; do
  python scripts/ab_fused.py $V 32768 20 2 tma:fused_impl=2 solo:fused_impl=4 > gpurun_out/ab_v${V}.log 2>&1
done
COPRIS_FUSED_IMPL=solo python scripts/trace_phases.py 32000 16384 > gpurun_out/trace_solo_32000.log 2>&1
COPRIS_FUSED_IMPL=solo TRACE_WARMUP=1 python scripts/trace_phases.py 32000 2048 > gpurun_out/trace_solo_32000_2048.log 2>&1
COPRIS_FUSED_IMPL=tma TRACE_WARMUP=1 python scripts/trace_phases.py 32000 2048 > gpurun_out/trace_tma_32000_2048.log 2>&1
