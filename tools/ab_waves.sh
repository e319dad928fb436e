# single-wave grids for the update (40 regs: 6 CTAs/SM = 888) and global-update (48 regs: 5/SM = 740) kernels
run() {
  echo "N=$1 $2 => $(env $2 timeout -s KILL 300 python bench.py --gpus $1 --skip-e2e --skip-cpu --skip-t1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); k=l["kernels"]; print(l["config"]["layout"], round(l["value"]), round(l["ms_per_step"],4), "upd", round(k["update"]["avg_ms"],4) if "update" in k else None)')"
}
for rep in 1 2; do
  run 1 "X=0"
  run 1 "LSGD_B200_UPD_CTAS=888"
  run 4 "X=0"
  run 4 "LSGD_B200_UPD_CTAS=888 LSGD_B200_GLOBAL_CTAS=740"
done
