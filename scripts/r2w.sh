for pdl in 0 1; do for gs in 1 10; do
COPRIS_PDL=$pdl timeout 300 python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --graph-steps $gs --no-e2e --no-cpu-baseline > gpurun_out/w_1x8_pdl${pdl}_gs${gs}.log 2>&1
done; done
COPRIS_PDL=1 timeout 300 python bench.py --config grpo_1x8_v32000_L256 --steps 300 --no-e2e --no-cpu-baseline > gpurun_out/w_1x8_pdl1_eager.log 2>&1
COPRIS_PDL=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/w_bench_pdl1.log 2>&1
COPRIS_PDL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_lmhead.py -q -m gpu --tb=short > gpurun_out/gpu_tests_w.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_w.log
