#!/bin/bash
# BASELINE.json configs[4]: vocab 32,000 short-response sweep on 1 GPU.
# 128 x 8 prompts (fills the GPU) and 1 x 8 (one group: launch + reduction
# overhead) at fixed lengths 256 .. 4096. One JSON line per run in
# $OUT/sweep_v32000.jsonl.
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
: > $OUT/sweep_v32000.jsonl
for L in 256 512 1024 2048 4096; do
  for P in 128 1; do
    steps=10; extra=""
    # one group: launch-bound, so the step is replayed as a CUDA graph
    [ $P = 1 ] && { steps=300; extra="--graph"; }
    timeout 300 python bench.py --config grpo_${P}x8_v32000_L$L --steps $steps --no-e2e \
      --no-cpu-baseline $extra "$@" 2>>$OUT/sweep_v32000.err | tail -1 >> $OUT/sweep_v32000.jsonl
  done
done
