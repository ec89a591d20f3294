for i in 1 2; do
COPRIS_LIB_PATH=$PWD/tmp_exp/old/libcopris_b200.so timeout 600 python bench.py --dlogits f32 --no-e2e --no-cpu-baseline > gpurun_out/v_f32_old_$i.log 2>&1
timeout 600 python bench.py --dlogits f32 --no-e2e --no-cpu-baseline > gpurun_out/v_f32_new_$i.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "dl_dtype1 or agree" --tb=short > gpurun_out/gpu_tests_v.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_v.log
COPRIS_BENCH_ONE_GPU=1 COPRIS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e > gpurun_out/v_rehearsal_torchrun.log 2>&1; echo rc=$? >> gpurun_out/v_rehearsal_torchrun.log
COPRIS_BENCH_ONE_GPU=1 COPRIS_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --config grpo_512x16_v151936 --steps 2 --warmup 3 --no-e2e > gpurun_out/v_rehearsal_self.log 2>&1; echo rc=$? >> gpurun_out/v_rehearsal_self.log
