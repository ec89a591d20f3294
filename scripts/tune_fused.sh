COPRIS_FUSED_IMPL=tma timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_tma.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_la2_3.log 2>&1
COPRIS_FUSED_IMPL=tma COPRIS_TUNE_CL=4 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_tma4.log 2>&1
