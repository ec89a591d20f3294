COPRIS_FUSED_IMPL=stream COPRIS_TUNE_WARPS=16 python scripts/trace_phases.py 151936 16384 > gpurun_out/trace_st16.log 2>&1
COPRIS_FUSED_IMPL=stream COPRIS_TUNE_WARPS=24 python scripts/trace_phases.py 151936 16384 > gpurun_out/trace_st24.log 2>&1
COPRIS_FUSED_IMPL=stream COPRIS_TUNE_WARPS=24 COPRIS_TUNE_SLOTS=3 python scripts/trace_phases.py 151936 16384 > gpurun_out/trace_st24s3.log 2>&1
python scripts/trace_phases.py 32000 65536 > gpurun_out/trace_tma32k.log 2>&1
