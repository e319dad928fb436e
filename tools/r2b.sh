# 4-GPU check: full GPU suite, bench.py --gpus N self-launched (no torchrun), flat CSGD beside it
set -x
nvidia-smi -L; nvidia-smi topo -m
timeout 1500 python -m pytest tests -m gpu -q -rA --timeout 900 > gpurun_out/r2b_pytest4.log 2>&1; echo pytest rc=$?
for n in 2 4; do
  timeout 600 python bench.py --gpus $n --skip-e2e > gpurun_out/r2b_bench_n$n.log 2>&1; echo bench n=$n rc=$?
  timeout 600 python bench.py --gpus $n --algo csgd --skip-e2e > gpurun_out/r2b_bench_csgd_n$n.log 2>&1; echo csgd n=$n rc=$?
done
timeout 600 python bench.py --gpus 4 --groups 4 --skip-e2e > gpurun_out/r2b_bench_4x1.log 2>&1; echo 4x1 rc=$?
timeout 600 python bench.py --gpus 4 --groups 1 --skip-e2e > gpurun_out/r2b_bench_1x4.log 2>&1; echo 1x4 rc=$?
tail -3 gpurun_out/r2b_pytest4.log
for f in gpurun_out/r2b_bench*.log; do echo $f; grep -o '"value": [0-9.]*, "unit": "samples/s", "n_gpus": [0-9]*, "steps": [0-9]*, "warmup": [0-9]*, "ms_per_step": [0-9.]*' $f; done
