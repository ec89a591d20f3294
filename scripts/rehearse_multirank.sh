# Control-flow rehearsal of bench.py's multi-rank path on ONE GPU (not a
# measurement): both ranks on cuda:0, gloo instead of NCCL (NCCL refuses two
# ranks on one device).
mkdir -p gpurun_out
export COPRIS_BENCH_ONE_GPU=1 COPRIS_BENCH_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/rehearse_weak.log 2>&1; echo "rc=$?" >> gpurun_out/rehearse_weak.log
timeout 600 python bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/rehearse_ref.log 2>&1; echo "rc=$?" >> gpurun_out/rehearse_ref.log
