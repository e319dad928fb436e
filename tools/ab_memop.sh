run() {
  echo "N=$1 $2 $3 => $(env $2 timeout -s KILL 300 python bench.py --gpus $1 $3 --skip-e2e --skip-cpu --skip-t1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["config"]["layout"], round(l["value"]), round(l["ms_per_step"],4))')"
}
timeout 1200 python -m pytest tests/test_gpu_ranks.py tests/test_gpu_parity.py -q -x -k "process_per_gpu or push_exchange or multi_gpu or sliced or jitter or missing_peer" 2>&1 | tail -2
for rep in 1 2; do
  run 4 "X=0"
  run 4 "LSGD_B200_SIGNAL_MEMOP=0"
  run 2 "X=0"
  run 2 "LSGD_B200_SIGNAL_MEMOP=0"
  run 4 "X=0" "--groups 4"
  run 4 "X=0" "--groups 1"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 tools/timeline.py --steps 3 --all-ranks > gpurun_out/r2_tl4m.txt 2>&1
