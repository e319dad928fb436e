# N=4 bench by LSGD layout (--groups): 1x4 (k=4, the 2x4 member count of N=8), 2x2 (default), 4x1
for rep in 1 2; do
  for g in 1 2 4; do
    echo "N4 groups=$g $(timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29760 + rep * 5 + g)) bench.py --gpus 4 --groups $g --skip-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"], l["config"]["layout"], round(l["step_roofline"]["frac"],3))')"
  done
done
