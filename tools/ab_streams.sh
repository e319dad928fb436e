# N=4 (2x2) bench by number of communicator streams, alternating on one box
for rep in 1 2; do
  for cfg in "4 2" "4 3" "4 4"; do
    set -- $cfg
    echo "N$1 comm_streams=$2 $(LSGD_B200_COMM_STREAMS=$2 timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 2959$rep bench.py --gpus $1 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
  done
done
LSGD_B200_COMM_STREAMS=4 timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/timeline.py --steps 2 > gpurun_out/timeline_n4_s4.txt 2> /dev/null
