COPRIS_FUSED_STREAM=1 COPRIS_TUNE_WARPS=16 python scripts/trace_phases.py 151936 16384 > gpurun_out/trace_st16.log 2>&1
COPRIS_FUSED_STREAM=1 COPRIS_TUNE_WARPS=8 python scripts/trace_phases.py 151936 16384 > gpurun_out/trace_st8.log 2>&1
COPRIS_FUSED_STREAM=1 COPRIS_TUNE_WARPS=8 python scripts/trace_phases.py 32000 65536 > gpurun_out/trace_st32k.log 2>&1
COPRIS_FUSED_STREAM=1 COPRIS_TUNE_WARPS=16 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "not fused_matches and not unfused and not padded" > gpurun_out/tune_tests.log 2>&1
