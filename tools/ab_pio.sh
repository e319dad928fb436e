run() {
  echo "N=$1 $2 => $(env $2 timeout -s KILL 300 python bench.py --gpus $1 --skip-cpu --skip-t1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); k=l["kernels"]; print(round(l["value"]), round(l["e2e"]["value"]) if l.get("e2e") else None, round(l["ms_per_step"],4), "gemm", round(k["gemm"]["ms_per_step"],4))')"
}
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -q -x -k "tc_training or weight_split or fp32_training or multi_gpu_matches or run_to_run" 2>&1 | tail -2
for rep in 1 2; do
for n in 1 2 4; do
  run $n "X=0"
  run $n "LSGD_B200_PREFETCH_IO=0"
done
done
