set -x
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
for V in 151936 32000; do
 for DL in bf16 f32; do
  $B --vocab $V --dlogits $DL --entropy-coeff 0.01 | sed "s/^/ENT_PAIR V=$V $DL /"
  COPRIS_FUSED_IMPL=1 $B --vocab $V --dlogits $DL --entropy-coeff 0.01 | sed "s/^/ENT_STREAM V=$V $DL /"
  $B --vocab $V --dlogits $DL | sed "s/^/NOENT V=$V $DL /"
 done
done
