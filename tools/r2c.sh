set -x
timeout 900 python -m pytest tests/test_gpu_ranks.py tests/test_gpu_parity.py -q -rA --timeout 600 -k "flat or nccl or hbm_weight or loss_history or missing_peer" > gpurun_out/r2c_pytest.log 2>&1; echo pytest rc=$?
timeout 300 python tools/mc_probe.py > gpurun_out/r2c_mc.log 2>&1
timeout 300 python tools/exchange_probe.py > gpurun_out/r2c_probe.jsonl 2> gpurun_out/r2c_probe.err; echo probe rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none --csv python tools/exchange_probe.py --reps 1 > gpurun_out/r2c_probe_ncu.csv 2> gpurun_out/r2c_probe_ncu.err; echo ncu rc=$?
for n in 2 4; do
  timeout 600 python bench.py --gpus $n --skip-e2e > gpurun_out/r2c_bench_n$n.log 2>&1; echo bench n=$n rc=$?
  timeout 600 python bench.py --gpus $n --algo csgd --skip-e2e > gpurun_out/r2c_bench_csgd_n$n.log 2>&1; echo csgd n=$n rc=$?
done
tail -3 gpurun_out/r2c_pytest.log; cat gpurun_out/r2c_mc.log; cat gpurun_out/r2c_probe.jsonl
