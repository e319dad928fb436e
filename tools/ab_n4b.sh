run() {
  echo "N=$1 $2 $3 => $(env $2 timeout -s KILL 300 python bench.py --gpus $1 $3 --skip-e2e --skip-t1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["config"]["layout"], round(l["value"]), round(l["ms_per_step"],4))')"
}
for rep in 1 2; do
  run 4 "X=0"
  run 4 "LSGD_B200_L0_DIV=1"
  run 4 "LSGD_B200_L0_DIV=4"
  run 4 "LSGD_B200_BUCKET_ELEMS=25165824"
  run 4 "LSGD_B200_BUCKET_ELEMS=50331648 LSGD_B200_GEMM_ELEMS=100663296"
  run 4 "LSGD_B200_GEMM_ELEMS=134217728"
  run 2 "X=0"
  run 2 "LSGD_B200_BUCKET_ELEMS=50331648"
  run 2 "LSGD_B200_L0_DIV=4"
  run 2 "LSGD_B200_BWD_ORDER=reverse"
done
