# full GPU check (under gpurun, 1 GPU): tests, smoke, bench lines for every
# BASELINE config, the reference arm, profiles. Logs in gpurun_out/.
timeout 1500 python -m pytest tests -q -m gpu --tb=short > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --dlogits f32 --no-e2e --no-cpu-baseline > gpurun_out/bench_f32.log 2>&1
timeout 300 python bench.py --config grpo_128x8_v151936_longtail_4stage --no-e2e --no-cpu-baseline > gpurun_out/bench_longtail.log 2>&1
timeout 600 python bench.py --config grpo_512x16_v151936 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_512x16.log 2>&1
timeout 300 python bench.py --config grpo_128x8_v32000_L256 --no-e2e --no-cpu-baseline > gpurun_out/bench_v32000.log 2>&1
timeout 300 python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --no-e2e --no-cpu-baseline > gpurun_out/bench_1x8_graph.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 oracle/_ref/trainer_loop_check 50 > gpurun_out/trainer_loop.jsonl 2> gpurun_out/trainer_loop.err
bash profiles/run_profile_r02.sh
python profiles/summarize.py r02 gpurun_out gpurun_out/profiles_r02 > gpurun_out/summarize.log 2>&1
rm -f gpurun_out/*.ncu-rep
