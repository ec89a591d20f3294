mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --tb=short > gpurun_out/full_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/full_gpu_tests.log
: > gpurun_out/san_summary.txt
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 0 --print-limit 50 --log-file gpurun_out/san_$tool.txt \
    python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused_reduction or claim_counter or graph or pair_rows or masked_vocabulary" -p no:cacheprovider \
    > gpurun_out/san_${tool}_pytest.txt 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/san_${tool}_pytest.txt)" >> gpurun_out/san_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/san_$tool.txt | tail -3 >> gpurun_out/san_summary.txt
done
python __graft_entry__.py smoke > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke2.log
