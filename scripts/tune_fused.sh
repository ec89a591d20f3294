timeout 900 python -m pytest tests -q -m gpu --tb=short -x 2>&1 | tail -5 > gpurun_out/la_tests.log
timeout 300 python scripts/micro/power_probe.py > gpurun_out/power.log 2>&1
python scripts/trace_phases.py 151936 16384 > gpurun_out/la2.log 2>&1
