set -x
timeout 2000 python -m pytest tests -m gpu -q -rA --timeout 900 > gpurun_out/r2s_pytest4.log 2>&1; echo pytest rc=$?
for n in 2 4; do
  timeout 600 python bench.py --gpus $n > gpurun_out/r2s_bench_n$n.log 2>&1; echo bench n=$n rc=$?
  timeout 600 python bench.py --gpus $n --algo csgd > gpurun_out/r2s_bench_csgd_n$n.log 2>&1; echo csgd n=$n rc=$?
done
timeout 600 python bench.py --gpus 4 --groups 4 --skip-e2e > gpurun_out/r2s_bench_4x1.log 2>&1
timeout 600 python bench.py --gpus 4 --groups 1 --skip-e2e > gpurun_out/r2s_bench_1x4.log 2>&1
timeout 600 python bench.py --gpus 4 --impl reference > gpurun_out/r2s_ref_n4.log 2>&1; echo ref rc=$?
tail -2 gpurun_out/r2s_pytest4.log; grep -E "^(FAILED|ERROR)" gpurun_out/r2s_pytest4.log
for f in gpurun_out/r2s_bench*.log; do echo "$f $(tail -1 $f | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["config"]["layout"], l["config"]["algorithm"], round(l["value"]), round(l["ms_per_step"],4), (l.get("e2e") or {}).get("value"), (l.get("exposed_comm") or {}).get("ms_per_step"))')"; done
