# N=4 (2x2) bench by exchange-kernel grid cap (LSGD_B200_COMM_CTAS), alternating on one box
for rep in 1 2; do
  for c in 148 296 592 74; do
    echo "N4 comm_ctas=$c $(LSGD_B200_COMM_CTAS=$c timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29950 + rep * 4 + c % 7)) bench.py --gpus 4 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
  done
done
