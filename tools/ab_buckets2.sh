# bench by exchange bucket / GEMM block size, alternating, on one box (N=2: 2x1, N=4: 2x2)
M=1048576
for rep in 1 2; do
  for cfg in "4 32 64" "4 32 128" "4 64 64" "2 32 32" "2 32 64" "2 16 64" "2 64 64"; do
    set -- $cfg
    echo "N$1 bucket=${2}M gemm=${3}M $(LSGD_B200_BUCKET_ELEMS=$(($2*M)) LSGD_B200_GEMM_ELEMS=$(($3*M)) timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 2958$rep bench.py --gpus $1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
  done
done
