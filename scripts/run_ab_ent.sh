# A/B: entropy pass 2 with folded constants (new, in-tree) vs tmp_exp/libold.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "entropy or kl" > gpurun_out/abent_tests.log 2>&1; echo "rc=$?" >> gpurun_out/abent_tests.log
summ() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); c=d['clocks']
        print(round(d['value']/1e6,3),'Mtok/s',d['config']['kernel']['kernel'],round(d['roofline']['frac'],4),c['sm_mhz'],c['reasons'])"; }
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --entropy-coeff 0.01"
{
for V in 151936 32000; do for DL in bf16 f32; do for rep in 1 2; do
  echo -n "OLD V=$V $DL: "; COPRIS_LIB_PATH=tmp_exp/libold.so $B --vocab $V --dlogits $DL 2>/dev/null | summ
  echo -n "NEW V=$V $DL: "; $B --vocab $V --dlogits $DL 2>/dev/null | summ
done; done; done
} > gpurun_out/ab_ent_fold.txt 2>&1
