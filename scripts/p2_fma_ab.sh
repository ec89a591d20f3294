# A/B of pair_p2_fma (pass-2 exponentials of the two-exponential modes partly on
# the FMA pipe): parity with the option on, then bench lines per mode, interleaved.
mkdir -p gpurun_out
COPRIS_PAIR_P2_FMA=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "entropy or f32 or F32 or masked or pair or kl or dropin or saturated" > gpurun_out/p2fma_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p2fma_tests.log
COPRIS_PAIR_P2_FMA=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "entropy or masked" > gpurun_out/p2fma4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p2fma4_tests.log
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
summ() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); c=d['clocks']
        print(round(d['value']/1e6,3),'Mtok/s',d['config']['kernel']['kernel'],round(d['roofline']['frac'],3),c['sm_mhz'],c['reasons'])"; }
for V in 151936 32000; do
 for MODE in "ent bf16" "ent f32" "noent f32"; do
  set -- $MODE
  EXTRA="--dlogits $2"; [ "$1" = ent ] && EXTRA="$EXTRA --entropy-coeff 0.01"
  for F in 0 1 2 3 0 2; do
   echo -n "V=$V $MODE p2_fma=$F "; COPRIS_PAIR_P2_FMA=$F $B --vocab $V $EXTRA 2>/dev/null | summ
  done
 done
done > gpurun_out/p2fma_ab.txt 2>&1
