for i in 1 2; do COPRIS_LMHEAD_GROUP=16 timeout 120 python scripts/bench_lmhead.py 4096 >> gpurun_out/lmb.log 2>&1; done
COPRIS_LMHEAD_GROUP=16 timeout 600 ncu --set full --import-source on -k regex:lmhead_fwd_pair -c 1 -o gpurun_out/lmhead_pair python scripts/bench_lmhead.py 4096 > /dev/null 2>&1
