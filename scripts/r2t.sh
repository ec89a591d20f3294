timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu --tb=short > gpurun_out/gpu_tests_t.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_t.log
for i in 1 2; do for b in 1 0; do
COPRIS_PAIR_BF16_STAGE=$b timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/t_bst${b}_$i.log 2>&1
done; done
for b in 1 0; do
COPRIS_PAIR_BF16_STAGE=$b timeout 300 python bench.py --config grpo_128x8_v32000_L256 --no-e2e --no-cpu-baseline > gpurun_out/t_v32k_bst${b}.log 2>&1
COPRIS_PAIR_BF16_STAGE=$b timeout 300 python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --no-e2e --no-cpu-baseline > gpurun_out/t_1x8_bst${b}.log 2>&1
done
