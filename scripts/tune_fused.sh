python scripts/trace_phases.py 151936 16384 > gpurun_out/trace_pf2.log 2>&1
cp paper_2511_05589_b200/libcopris_b200.so /tmp/keep.so; cp scripts/micro/lib_pf1.so paper_2511_05589_b200/libcopris_b200.so
python scripts/trace_phases.py 151936 16384 > gpurun_out/trace_pf1.log 2>&1
cp /tmp/keep.so paper_2511_05589_b200/libcopris_b200.so
