# Round-end measurement set on one 4-GPU box: bench N=1/2/4 (+ reference arm), N=4 timeline
python bench.py > gpurun_out/r1_bench_cfg3_n1.jsonl 2> gpurun_out/b1.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/r1_bench_cfg3_n2.jsonl 2> gpurun_out/b2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 > gpurun_out/r1_bench_cfg3_n4.jsonl 2> gpurun_out/b4.err
python bench.py --impl reference > gpurun_out/r1_bench_reference_n1.jsonl 2> gpurun_out/br.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 tools/timeline.py --steps 2 > gpurun_out/r1_timeline_n4.txt 2> gpurun_out/t4.err
