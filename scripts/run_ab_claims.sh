# A/B: first row's loads before the initial row claims (new, in-tree) vs tmp_exp/libold.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py -q -x > gpurun_out/abcl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/abcl_tests.log
summ() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); c=d['clocks']
        print(round(d['value']/1e6,3),'Mtok/s',round(d['ms_per_step'],4),'ms',d['config']['kernel']['kernel'],round(d['roofline']['frac'],4),c['sm_mhz'],c['reasons'])"; }
sw() { python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['rows'], round(d['us_per_step'],2), round(d['frac'],3))"; }
{
for rep in 1 2; do
  echo "OLD sweep:"; COPRIS_LIB_PATH=tmp_exp/libold.so python scripts/small_step_sweep.py solo 2>&1 | sw
  echo "NEW sweep:"; python scripts/small_step_sweep.py solo 2>&1 | sw
done
for rep in 1 2 3; do
  echo -n "OLD 1x8 graph: "; COPRIS_LIB_PATH=tmp_exp/libold.so python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --no-e2e --no-cpu-baseline 2>/dev/null | summ
  echo -n "NEW 1x8 graph: "; python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --no-e2e --no-cpu-baseline 2>/dev/null | summ
done
for rep in 1 2; do
  echo -n "OLD 1x8 v151936 graph: "; COPRIS_LIB_PATH=tmp_exp/libold.so python bench.py --config grpo_1x8_v32000_L256 --vocab 151936 --steps 100 --graph --no-e2e --no-cpu-baseline 2>/dev/null | summ
  echo -n "NEW 1x8 v151936 graph: "; python bench.py --config grpo_1x8_v32000_L256 --vocab 151936 --steps 100 --graph --no-e2e --no-cpu-baseline 2>/dev/null | summ
  echo -n "OLD cfg2: "; COPRIS_LIB_PATH=tmp_exp/libold.so python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | summ
  echo -n "NEW cfg2: "; python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | summ
done
} > gpurun_out/ab_claims.txt 2>&1
