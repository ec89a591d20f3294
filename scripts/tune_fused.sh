timeout 600 env COPRIS_TUNE_P2G=1 python -m pytest tests/test_gpu_parity.py -x -q --tb=short -k "stream or 151936" 2>&1 | tail -3 > gpurun_out/t.log
for v in 0 1; do COPRIS_TUNE_P2G=$v python scripts/trace_phases.py 151936 16384 > gpurun_out/p2g$v.log 2>&1; done
PROBE_VARIANTS=stream:2 timeout 300 python scripts/micro/power_probe.py > gpurun_out/power0.log 2>&1
COPRIS_TUNE_P2G=1 PROBE_VARIANTS=stream:2 timeout 300 python scripts/micro/power_probe.py > gpurun_out/power1.log 2>&1
