mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for V in 151936 32000; do python scripts/cta_tail.py $V 32768 2 | cut -c1-260; COPRIS_PAIR_DYNAMIC=0 python scripts/cta_tail.py $V 32768 1 | sed 's/^/STATIC /' | cut -c1-260; done
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for k in 1 2; do
 for D in 1 0; do
  COPRIS_PAIR_DYNAMIC=$D $B | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('DYN=$D', 'V151936', round(j['value']/1e6,3), round(j['roofline']['frac'],4), j['clocks'].get('sm_mhz'), j['clocks'].get('reasons'))"
  COPRIS_PAIR_DYNAMIC=$D $B --vocab 32000 | python -c "import sys,json; j=json.loads(sys.stdin.read()); print('DYN=$D', 'V32000', round(j['value']/1e6,3), round(j['roofline']['frac'],4), j['clocks'].get('sm_mhz'), j['clocks'].get('reasons'))"
 done
done
