run() {
  echo "N=$1 $2 => $(env $2 timeout -s KILL 300 python bench.py --gpus $1 --skip-e2e --skip-cpu --skip-t1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); k=l["kernels"]; print(round(l["value"]), round(l["ms_per_step"],4), "gemm", round(k["gemm"]["ms_per_step"],4))')"
}
for rep in 1 2; do
for n in 1 4; do
  run $n "X=0"
  run $n "LSGD_B200_UPD_CTAS=1036 LSGD_B200_GLOBAL_CTAS=1036"
  run $n "LSGD_B200_UPD_CTAS=4000000 LSGD_B200_GLOBAL_CTAS=4000000"
  run $n "LSGD_B200_UPD_CTAS=4000000 LSGD_B200_GLOBAL_CTAS=4000000 LSGD_B200_COMM_CTAS=4000000"
  run $n "LSGD_B200_UPD_CTAS=2368 LSGD_B200_GLOBAL_CTAS=2368"
done
done
