# side-kernel footprint A/B at N=4 (2x2) and N=2 (2x1): grids and SM exclusion of the exchange / update kernels
run() {
  echo "N=$1 $2 => $(env $2 timeout -s KILL 300 python bench.py --gpus $1 --skip-e2e --skip-t1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), round(l["ms_per_step"],4))')"
}
for rep in 1 2; do
for n in 4 2; do
  run $n "X=0"
  run $n "LSGD_B200_SIDE_SMEM=24576"
  run $n "LSGD_B200_UPD_CTAS=296 LSGD_B200_GLOBAL_CTAS=296"
  run $n "LSGD_B200_UPD_CTAS=592 LSGD_B200_GLOBAL_CTAS=592"
  run $n "LSGD_B200_GLOBAL_CTAS=296"
  run $n "LSGD_B200_UPD_CTAS=296"
  run $n "LSGD_B200_COMM_CTAS=74"
  run $n "LSGD_B200_UPD_CTAS=148 LSGD_B200_GLOBAL_CTAS=148 LSGD_B200_COMM_CTAS=74"
done
done
