run() {
  echo "$1 => $(env $1 timeout -s KILL 300 python bench.py --skip-e2e --skip-cpu 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), round(l["ms_per_step"],4), round(l["kernels"]["gemm"]["ms_per_step"],4))')"
}
for rep in 1 2 3; do
for v in "X=0" "LSGD_B200_BUCKET_ELEMS=33554432" "LSGD_B200_BUCKET_ELEMS=50331648" "LSGD_B200_BUCKET_ELEMS=67108864" "LSGD_B200_BUCKET_ELEMS=33554432 LSGD_B200_UPD_UNROLL=2" "LSGD_B200_BUCKET_ELEMS=25165824"; do
  run "$v"
done
done
