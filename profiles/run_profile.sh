#!/bin/bash
# Profiling recipe (run under gpurun, 1 GPU; B200_PROFILING.md):
#   1. launch list of the bench command (cold, serialised: compare SHARES)
#   2. one `ncu --set full` capture of the fused kernel (and the unfused K3)
# Outputs land in gpurun_out/; summaries are copied into profiles/ by hand.
set -u
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_ -s 3 -c 1 \
    -o $OUT/prof_fused -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --chunk-rows 8192 > $OUT/prof_fused.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_tma -s 2 -c 1 \
    -o $OUT/prof_tma -f \
    python bench.py --config grpo_128x8_v32000_L1024 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    --chunk-rows 16384 > $OUT/prof_tma.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|fused_stream" -s 2 -c 2 \
    -o $OUT/prof_unfused -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --chunk-rows 8192 --unfused > $OUT/prof_unfused.log 2>&1
COPRIS_LMHEAD_GROUP=16 ncu --set full --clock-control none --import-source on -k regex:lmhead_fwd_pair -c 1 \
    -o $OUT/prof_lmhead -f python scripts/bench_lmhead.py 4096 > $OUT/prof_lmhead.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lmhead_fwd_pair -c 1 \
    -o $OUT/prof_lmhead_dw -f python scripts/bench_lmhead_dw.py 4096 > $OUT/prof_lmhead_dw.log 2>&1
