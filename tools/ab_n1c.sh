run() {
  echo "$1 => $(env $1 timeout -s KILL 300 python bench.py --skip-e2e --skip-cpu 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); k=l["kernels"]; print(round(l["value"]), round(l["ms_per_step"],4), "gemm", round(k["gemm"]["ms_per_step"],4))')"
}
timeout 300 python tools/timeline.py --steps 3 > gpurun_out/r2_tl1_64m.txt 2>&1
for rep in 1 2; do
for v in "X=0" "LSGD_B200_BWD_SEQ=x2,x1,w1.0,w0,w1.1,w2" "LSGD_B200_BWD_SEQ=x2,w2,x1,w0,w1" "LSGD_B200_BWD_SEQ=x2,x1,w1,w0,w2" "LSGD_B200_BWD_SEQ=x2,w1.0,x1,w0,w1.1,w2" "LSGD_B200_BWD_SEQ=w2,x2,w1,x1,w0"; do
  run "$v"
done
done
