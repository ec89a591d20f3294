timeout 600 python bench.py > gpurun_out/u_bench.log 2>&1
bash profiles/run_profile_r02.sh
python profiles/summarize.py r02 gpurun_out gpurun_out/profiles_r02 > gpurun_out/summarize.log 2>&1
rm -f gpurun_out/*.ncu-rep
timeout 300 python bench.py --config grpo_1x8_v32000_L256 --steps 300 --graph --no-e2e --no-cpu-baseline > gpurun_out/u_1x8.log 2>&1
timeout 300 python bench.py --config grpo_128x8_v32000_L256 --no-e2e --no-cpu-baseline > gpurun_out/u_128_v32k.log 2>&1
timeout 300 python bench.py --config grpo_128x8_v151936_longtail_4stage --no-e2e --no-cpu-baseline > gpurun_out/u_longtail.log 2>&1
timeout 600 python bench.py --config grpo_512x16_v151936 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/u_512x16.log 2>&1
timeout 600 python bench.py --dlogits f32 --no-e2e --no-cpu-baseline > gpurun_out/u_f32.log 2>&1
