# what the round-end driver runs on one fresh B200: the GPU suite, smoke(), both bench arms
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/dl_pytest.log 2>&1; echo pytest rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dl_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/dl_ref.log 2>&1; echo ref rc=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/dl_bench.log 2>&1; echo bench rc=$?
tail -2 gpurun_out/dl_pytest.log; tail -1 gpurun_out/dl_smoke.log; tail -c 400 gpurun_out/dl_ref.log; echo; tail -c 2500 gpurun_out/dl_bench.log
