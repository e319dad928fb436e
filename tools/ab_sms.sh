# bench by GEMM grid cap (LSGD_TC_MAX_SMS), alternating on one box
for rep in 1 2; do
  for v in 128 148 136; do
    echo "N1 max_sms=$v $(LSGD_TC_MAX_SMS=$v timeout -s KILL 300 python bench.py --skip-cpu --skip-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
    echo "N4 max_sms=$v $(LSGD_TC_MAX_SMS=$v timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + rep * 7 + v % 5)) bench.py --gpus 4 --skip-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
  done
done
