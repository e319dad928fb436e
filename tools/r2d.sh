set -x
timeout 200 python tools/nvml_probe.py > gpurun_out/r2d_nvml.log 2>&1
for n in 4 2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29555 tools/timeline.py --steps 3 > gpurun_out/r2d_timeline_n$n.txt 2>gpurun_out/r2d_timeline_n$n.err; echo tl rc=$?
done
timeout 600 python bench.py --gpus 4 --skip-e2e > gpurun_out/r2d_bench_n4.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --gpus 4 --algo csgd --skip-e2e > gpurun_out/r2d_bench_csgd_n4.log 2>&1; echo bench rc=$?
cat gpurun_out/r2d_nvml.log
