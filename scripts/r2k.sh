for i in 1 2; do for st in 1 0; do
COPRIS_PAIR_ST256=$st timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/k_st${st}_$i.log 2>&1
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --tb=short > gpurun_out/gpu_tests_k.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_k.log
