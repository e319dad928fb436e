run() {
  echo "$1 => $(env $1 timeout -s KILL 300 python bench.py --skip-e2e --skip-cpu 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); k=l["kernels"]; print(round(l["value"]), round(l["ms_per_step"],4), "gemm", round(k["gemm"]["ms_per_step"],4), "upd", round(k["update"]["avg_ms"],4))')"
}
for rep in 1 2; do
for v in "X=0" "LSGD_B200_UPD_CTAS=296 LSGD_B200_UPD_UNROLL=2" "LSGD_B200_UPD_CTAS=296 LSGD_B200_UPD_UNROLL=4" "LSGD_B200_UPD_CTAS=148 LSGD_B200_UPD_UNROLL=4" "LSGD_B200_UPD_CTAS=592 LSGD_B200_UPD_UNROLL=2" "LSGD_B200_UPD_CTAS=296"; do
  run "$v"
done
done
