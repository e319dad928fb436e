# backward op order A/B (LSGD_B200_BWD_SEQ) at N=2 (2x1) and N=4 (2x2), one box, bench.py self-launched
run() {  # $1 = N, $2 = env assignments
  echo "N=$1 $2 => $(env $2 timeout -s KILL 300 python bench.py --gpus $1 --skip-e2e --skip-t1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), round(l["ms_per_step"],4))')"
}
for rep in 1 2; do
  run 2 "X=0"
  run 2 "LSGD_B200_BWD_SEQ=w2,x2,w1,x1,w0"
  run 2 "LSGD_B200_BWD_SEQ=x2,w1.0,x1,w0,w1.1,w2"
  run 2 "LSGD_B200_BWD_SEQ=x2,w1,x1,w0,w2"
  run 2 "LSGD_B200_BWD_SEQ=x2,x1,w0.0,w1.0,w0.1,w1.1,w2"
  run 2 "LSGD_B200_BWD_SEQ=x2,w1.0,x1,w0.0,w1.1,w0.1,w2"
  run 4 "X=0"
  run 4 "LSGD_B200_BWD_SEQ=x2,w1,x1,w0,w2"
  run 4 "LSGD_B200_GEMM_ELEMS=33554432 LSGD_B200_BWD_SEQ=x2,w1.0,x1,w0,w1.1,w2"
  run 4 "LSGD_B200_GEMM_ELEMS=33554432 LSGD_B200_BWD_SEQ=w2,x2,w1.0,w1.1,x1,w0"
  run 4 "LSGD_B200_GEMM_ELEMS=33554432 LSGD_B200_BWD_SEQ=x2,w1.0,x1,w0.0,w1.1,w0.1,w2"
done
