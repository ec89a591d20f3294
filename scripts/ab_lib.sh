# A/B of two builds of the library on one box, interleaved: the in-tree build
# (new) against tmp_exp/libold.so (old). Usage: bash scripts/ab_lib.sh [bench args...]
mkdir -p gpurun_out
summ() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); c=d['clocks']
        print(round(d['value']/1e6,3),'Mtok/s',d['config']['kernel']['kernel'],round(d['roofline']['frac'],4),c['sm_mhz'],c.get('power_w'),c['reasons'])"; }
B="python bench.py --no-e2e --no-cpu-baseline"
for cfg in "" "--vocab 32000" "--dlogits f32"; do
 for rep in 1 2 3; do
  echo -n "OLD $cfg: "; COPRIS_LIB_PATH=tmp_exp/libold.so $B $cfg 2>/dev/null | summ
  echo -n "NEW $cfg: "; $B $cfg 2>/dev/null | summ
 done
done
