set -x
timeout 900 python -m pytest tests/test_gpu_ranks.py tests/test_gpu_parity.py -q -rA --timeout 600 -k "sliced or push_exchange or replicas or multi_gpu_matches or process_per_gpu" > gpurun_out/r2i_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r2i_pytest.log
for g in 4 2 1; do
  timeout 300 python bench.py --gpus 4 --groups $g --skip-e2e --skip-t1 > gpurun_out/r2i_bench_g$g.log 2>&1; echo g=$g rc=$?
done
LSGD_B200_SLICED_GLOBAL=1 timeout 300 python bench.py --gpus 4 --groups 2 --skip-e2e --skip-t1 > gpurun_out/r2i_bench_g2_sliced.log 2>&1
LSGD_B200_SLICED_GLOBAL=0 timeout 300 python bench.py --gpus 4 --groups 4 --skip-e2e --skip-t1 > gpurun_out/r2i_bench_g4_whole.log 2>&1
for f in gpurun_out/r2i_bench*.log; do echo "$f $(tail -1 $f | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["config"]["layout"], round(l["value"]), round(l["ms_per_step"],4))')"; done
