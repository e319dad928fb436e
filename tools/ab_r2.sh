# A/B of schedule knobs at N=4 (2x2), one box, bench.py self-launched; prints value and ms/step per variant
run() {
  echo "$1 => $(env $1 timeout -s KILL 300 python bench.py --gpus 4 --skip-e2e --skip-t1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), round(l["ms_per_step"],4))')"
}
for rep in 1 2; do
for v in "X=0" "LSGD_TC_MAX_SMS=120" "LSGD_TC_MAX_SMS=112" "LSGD_TC_MAX_SMS=96" "LSGD_B200_DMA=7" "LSGD_B200_DMA=11" "LSGD_B200_COMM_CTAS=296" "LSGD_B200_BWD_ORDER=dx_first" "LSGD_B200_COMM_STREAMS=2"; do
  run "$v"
done
done
