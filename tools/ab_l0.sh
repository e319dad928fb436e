# N=4 (2x2) and N=2 (2x1) bench by layer-0 bucket divisor (LSGD_B200_L0_DIV), alternating on one box
for rep in 1 2; do
  for cfg in "4 2" "4 4" "4 1" "2 2" "2 4"; do
    set -- $cfg
    echo "N$1 l0_div=$2 $(LSGD_B200_L0_DIV=$2 timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29850 + rep * 10 + $1 + $2)) bench.py --gpus $1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
  done
done
