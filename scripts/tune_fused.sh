for k in 2 4 8; do COPRIS_TUNE_K=$k python scripts/trace_phases.py 151936 16384 > gpurun_out/trace_k$k.log 2>&1; done
COPRIS_TUNE_K=8 COPRIS_TUNE_SLOTS=2 python scripts/trace_phases.py 151936 16384 > gpurun_out/trace_k8s2.log 2>&1
COPRIS_TUNE_K=2 COPRIS_TUNE_SLOTS=12 python scripts/trace_phases.py 151936 16384 > gpurun_out/trace_k2s12.log 2>&1
