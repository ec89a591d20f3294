timeout 1500 python -m pytest tests -q -m gpu --tb=short > gpurun_out/gpu_tests_q.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_q.log
python __graft_entry__.py smoke > gpurun_out/smoke_q.log 2>&1
timeout 600 python bench.py > gpurun_out/q_bench.log 2>&1
timeout 300 python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --no-e2e --no-cpu-baseline > gpurun_out/q_1x8.log 2>&1
timeout 300 python bench.py --config grpo_128x8_v32000_L256 --no-e2e --no-cpu-baseline > gpurun_out/q_128_v32k.log 2>&1
timeout 300 python bench.py --config grpo_128x8_v151936_longtail_4stage --no-e2e --no-cpu-baseline > gpurun_out/q_longtail.log 2>&1
timeout 600 python bench.py --config grpo_512x16_v151936 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q_512x16.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/q_ref.log 2>&1
