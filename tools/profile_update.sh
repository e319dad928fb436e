# ncu --set full of the K8 update kernel on the cfg4 synthetic-gradient step (one GPU; the plain command first)
CMD="python bench.py --workload cfg4 --steps 2 --warmup 3 --skip-cpu --skip-e2e"
$CMD > gpurun_out/prof_upd_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:update_kernel -s 3 -c 2 -o gpurun_out/prof_update $CMD \
  > gpurun_out/ncu_update.log 2>&1
echo "profile rc=$?" >> gpurun_out/ncu_update.log
ncu -i gpurun_out/prof_update.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size > gpurun_out/ncu_update.csv 2>&1
