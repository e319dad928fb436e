set -x
ev() {
  echo "$1 $2 => $(env $1 timeout -s KILL 300 python bench.py --gpus 4 --skip-t1 $2 2>/dev/null | tail -1 | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["config"]["layout"], round(l["value"]), round(l["e2e"]["value"]) if l.get("e2e") else None, round(l["ms_per_step"],4))')"
}
for rep in 1 2; do
  ev "X=0"
  ev "LSGD_B200_DMA=1"
  ev "LSGD_B200_DMA=0"
done
for n in 1 2 4; do
  timeout 300 python bench.py --gpus $n --workload cfg4 --skip-cpu > gpurun_out/r2x_cfg4_n$n.log 2>&1; echo cfg4 n=$n rc=$?
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29577 sweep.py --sizes 20,22,24,26,28 > gpurun_out/r2x_sweep_n4.jsonl 2> gpurun_out/r2x_sweep_n4.err; echo sweep rc=$?
for f in gpurun_out/r2x_cfg4_n*.log; do tail -1 $f | cut -c1-400; done
cat gpurun_out/r2x_sweep_n4.jsonl | cut -c1-300
