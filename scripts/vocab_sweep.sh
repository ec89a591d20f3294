# Vocabulary sweep of the default kernels at config #2's batch shape (128 x 8,
# lognormal lengths up to 8k): common model vocabularies, bf16 dlogits.
OUT=${OUT:-gpurun_out}
for V in 32000 32768 50304 65536 100352 128256 151936 152064 200064 229376 256000; do
  timeout 600 python bench.py --vocab $V --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/vsweep_$V.log 2>&1
done
