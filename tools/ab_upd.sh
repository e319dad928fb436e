# N=4 (2x2) bench by update-kernel grid cap / unroll, one box
for cfg in "1184 1" "296 1" "592 1" "1184 2" "1184 1"; do
  set -- $cfg
  echo "N4 upd_ctas=$1 unroll=$2 $(LSGD_B200_UPD_CTAS=$1 LSGD_B200_UPD_UNROLL=$2 timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29400 + $1 % 97 + $2)) bench.py --gpus 4 --skip-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
done
