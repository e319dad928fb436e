# bench by backward order (LSGD_B200_BWD_ORDER), alternating on one box
for rep in 1 2; do
  for cfg in "4 reverse" "4 dx_first" "2 reverse" "2 dx_first"; do
    set -- $cfg
    echo "N$1 order=$2 $(LSGD_B200_BWD_ORDER=$2 timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 2960$rep bench.py --gpus $1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
  done
done
