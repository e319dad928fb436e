# bench with the bias gradient on its own stream (default) vs on the main stream, alternating on one box
for rep in 1 2; do
  for bs in 1 0; do
    echo "N1 bias_stream=$bs $(LSGD_B200_BIAS_STREAM=$bs timeout -s KILL 300 python bench.py --skip-cpu 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
    echo "N4 bias_stream=$bs $(LSGD_B200_BIAS_STREAM=$bs timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800 + rep * 2 + bs)) bench.py --gpus 4 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
  done
done
