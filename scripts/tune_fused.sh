python scripts/trace_phases.py 32000 65536 > gpurun_out/trace_tma32k.log 2>&1
timeout 300 python bench.py --config grpo_128x8_v32000_L1024 --no-e2e --no-cpu-baseline > gpurun_out/bench_v32000.log 2>&1
