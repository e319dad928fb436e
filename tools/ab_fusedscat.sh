run() {
  echo "N=$1 $2 => $(env $2 timeout -s KILL 300 python bench.py --gpus $1 --skip-e2e --skip-cpu --skip-t1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["config"]["layout"], round(l["value"]), round(l["ms_per_step"],4))')"
}
for rep in 1 2; do
  run 4 "X=0"
  run 4 "LSGD_B200_DMA=1 LSGD_B200_GEMM_ELEMS=33554432"
  run 4 "LSGD_B200_GEMM_ELEMS=33554432"
done
