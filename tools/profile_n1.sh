# 1-GPU profiling recipe (B200_PROFILING.md): the plain command must exit 0 before ncu runs the same command.
#   1. launch list of every kernel of the bench command (cold-cache, serialised per-launch durations)
#   2. ncu --set full of one step's tensor-core GEMM launches (skip the 3 warm-up steps x 9 GEMMs: 64M buckets)
CMD="python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD \
  > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32x3 -s ${SKIP:-27} -c ${COUNT:-9} -o gpurun_out/prof_gemm $CMD \
  > gpurun_out/ncu_full.log 2>&1
echo "profile rc=$?" >> gpurun_out/ncu_full.log
