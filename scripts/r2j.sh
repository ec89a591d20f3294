for T in 4096 8192; do for i in 1 2; do
timeout 600 python scripts/bench_lmhead.py $T > gpurun_out/lmhead_${T}_$i.log 2>&1
done; done
for i in 1 2 3; do
ncu --set full --clock-control none -k regex:lmhead_fwd_pair -c 1 -o gpurun_out/prof_lmhead_$i -f python scripts/bench_lmhead.py 4096 > gpurun_out/prof_lmhead_$i.log 2>&1
ncu -i gpurun_out/prof_lmhead_$i.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum > gpurun_out/prof_lmhead_$i.csv 2>&1
done
rm -f gpurun_out/*.ncu-rep
