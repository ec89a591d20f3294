#!/bin/bash
# Round-2 profiling recipe (under gpurun, 1 GPU; B200_PROFILING.md): launch list
# of the default bench command, one `ncu --set full` capture of the default
# fused kernel at V = 151,936 (fused_pair_kernel) with bf16 and with f32
# dlogits. Outputs in gpurun_out/; summarised by profiles/summarize.py.
set -u
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_ -s 3 -c 1 \
    -o $OUT/prof_fused -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --chunk-rows 8192 > $OUT/prof_fused.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_ -s 3 -c 1 \
    -o $OUT/prof_fused_f32 -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --chunk-rows 8192 --dlogits f32 \
    > $OUT/prof_fused_f32.log 2>&1
# V = 32,000 (config #5): the solo kernel, 16,384-row launch
ncu --set full --clock-control none --import-source on -k regex:fused_ -s 3 -c 1 \
    -o $OUT/prof_tma -f \
    python bench.py --config grpo_128x8_v32000_L1024 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    --chunk-rows 16384 > $OUT/prof_tma.log 2>&1
