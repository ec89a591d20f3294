timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/ab_parity.log 2>&1; echo "rc=$?" >> gpurun_out/ab_parity.log
bash scripts/ab_lib.sh > gpurun_out/ab_target_prefetch.txt 2>&1
