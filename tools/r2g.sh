set -x
timeout 1800 python -m pytest tests -m gpu -q -rA --timeout 900 > gpurun_out/r2g_pytest4.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --gpus 4 --skip-e2e > gpurun_out/r2g_bench_n4.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --gpus 2 --skip-e2e > gpurun_out/r2g_bench_n2.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/r2g_pytest4.log; grep -E "FAIL|Error" gpurun_out/r2g_pytest4.log | head
