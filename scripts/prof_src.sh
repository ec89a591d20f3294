mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:fused_ -s 3 -c 1 \
    -o gpurun_out/src_pair -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --chunk-rows 8192 > gpurun_out/src_pair.log 2>&1
ls -la gpurun_out/src_pair.ncu-rep
