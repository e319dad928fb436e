# Round-2 final measurements on one 4-GPU box: the GPU suite, bench.py at N = 1, 2, 4 (LSGD and flat CSGD), layouts,
# the reference arm at N = 1 and 4, a per-rank N = 4 timeline
set -x
timeout 1800 python -m pytest tests -m gpu -q -rA --timeout 900 > gpurun_out/f_pytest4.log 2>&1; echo pytest rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/f_bench_n1.log 2>&1; echo n1 rc=$?
for n in 2 4; do
  timeout 600 python bench.py --gpus $n > gpurun_out/f_bench_n$n.log 2>&1; echo n=$n rc=$?
  timeout 600 python bench.py --gpus $n --algo csgd > gpurun_out/f_bench_csgd_n$n.log 2>&1; echo csgd n=$n rc=$?
done
timeout 600 python bench.py --gpus 4 --groups 4 --skip-e2e > gpurun_out/f_bench_4x1.log 2>&1
timeout 600 python bench.py --gpus 4 --groups 1 --skip-e2e > gpurun_out/f_bench_1x4.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/f_ref_n1.log 2>&1; echo ref1 rc=$?
timeout 900 python bench.py --impl reference --gpus 4 > gpurun_out/f_ref_n4.log 2>&1; echo ref4 rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 tools/timeline.py --steps 3 --all-ranks > gpurun_out/f_timeline_n4.txt 2>&1
tail -2 gpurun_out/f_pytest4.log; grep -E "^(FAILED|ERROR)" gpurun_out/f_pytest4.log
for f in gpurun_out/f_bench*.log gpurun_out/f_ref*.log; do echo "$f $(tail -1 $f | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["config"].get("layout"), l["config"].get("algorithm"), round(l["value"],2), round(l["ms_per_step"],4) if "ms_per_step" in l else None, (l.get("e2e") or {}).get("value"), (l.get("exposed_comm") or {}).get("ms_per_step"))')"; done
