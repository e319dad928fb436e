# N=1 A/B: update-kernel footprint vs the weight-gradient GEMMs it overlaps
run() {
  echo "$1 => $(env $1 timeout -s KILL 300 python bench.py --skip-e2e --skip-cpu 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), round(l["ms_per_step"],4), round(l["kernels"]["gemm"]["ms_per_step"],4))')"
}
for rep in 1 2; do
for v in "X=0" "LSGD_B200_UPD_CTAS=148" "LSGD_B200_UPD_CTAS=296" "LSGD_B200_UPD_CTAS=592" "LSGD_B200_UPD_UNROLL=2" "LSGD_B200_UPD_UNROLL=4" "LSGD_B200_BUCKET_ELEMS=33554432" "LSGD_B200_BUCKET_ELEMS=8388608" "LSGD_B200_FUSED_UPDATE=1" "LSGD_B200_SIDE_SMEM=24576"; do
  run "$v"
done
done
