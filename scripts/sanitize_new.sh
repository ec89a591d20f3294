#!/bin/bash
# compute-sanitizer over the GPU parity tests (every fused-kernel variant, the
# unfused K1/K2/K3 path, KL + entropy, token masks, CUDA-graph replay, the
# LM-head kernels, Adam, the host-buffer pipeline). Run under gpurun (1 GPU);
# reports in $OUT/sanitizer_<tool>.txt, summary lines in $OUT/sanitizer_summary.txt.
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
SEL=${SEL:-"dl_dtype0 or unfused or kl_and_entropy or loss_mask or graph or k1_equals or behaviour or reduce or determin"}
: > $OUT/sanitizer_summary.txt
for tool in memcheck synccheck; do
  timeout 3000 compute-sanitizer --tool $tool --error-exitcode 0 --print-limit 50 \
      --log-file $OUT/sanitizer_$tool.txt \
      python -m pytest tests/test_gpu_parity.py \
      -q -m gpu -x -k "$SEL" -p no:cacheprovider \
      > $OUT/sanitizer_${tool}_pytest.txt 2>&1
  echo "$tool pytest rc=$? $(tail -1 $OUT/sanitizer_${tool}_pytest.txt)" >> $OUT/sanitizer_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" $OUT/sanitizer_$tool.txt | tail -3 >> $OUT/sanitizer_summary.txt
done
