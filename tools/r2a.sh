set -x
nvidia-smi -L
timeout 1200 python -m pytest tests -m gpu -q -rA --timeout 600 > gpurun_out/r2a_pytest.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/r2a_bench.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/r2a_pytest.log; tail -2 gpurun_out/r2a_smoke.log; tail -c 3000 gpurun_out/r2a_bench.log
