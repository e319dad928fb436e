# N=4 (2x2) bench by copy-engine bit mask (LSGD_B200_DMA), 4 communicator streams, short timeouts (a hang is killed)
for rep in 1 2; do
  for d in 3 7 11 15; do
    echo "N4 dma=$d $(LSGD_B200_COMM_STREAMS=4 LSGD_B200_DMA=$d timeout -s KILL 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + rep * 20 + d)) bench.py --gpus 4 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])' 2>&1 | tail -1)"
  done
done
