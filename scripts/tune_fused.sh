python scripts/trace_phases.py 151936 16384 > gpurun_out/trace_emu.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "151936 or saturated or deterministic or kl" > gpurun_out/tune_tests.log 2>&1
