# A/B of the accumulation chunk on one box: bench.py at N=1 and N=4, alternating LSGD_TC_KCHUNK values
for rep in 1 2; do
  for kc in 512 0 1024; do
    echo "N1 kc=$kc $(LSGD_TC_KCHUNK=$kc timeout -s KILL 300 python bench.py 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
    echo "N4 kc=$kc $(LSGD_TC_KCHUNK=$kc timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2954$rep bench.py --gpus 4 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"]), l["ms_per_step"])')"
  done
done
