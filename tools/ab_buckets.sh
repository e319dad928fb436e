# N=4 (2x2) bench by exchange bucket / GEMM block size, alternating, on one box
M=1048576
for rep in 1 2; do
  for cfg in "64 64" "32 32" "32 64" "16 64" "24 24"; do
    set -- $cfg
    echo "N4 bucket=${1}M gemm=${2}M $(LSGD_B200_BUCKET_ELEMS=$(($1*M)) LSGD_B200_GEMM_ELEMS=$(($2*M)) timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2957$rep bench.py --gpus 4 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
  done
done
