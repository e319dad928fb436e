set -x
timeout 300 python tools/tf32_peak.py > gpurun_out/r2f_tf32.log 2>&1; echo tf32 rc=$?
timeout 900 python -m pytest tests/test_gpu_tc.py -q -rA --timeout 800 -k "cfg3_steps_match_reference" -s > gpurun_out/r2f_cfg3.log 2>&1; echo cfg3 rc=$?
timeout 900 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_exchange.py > gpurun_out/r2f_synccheck.log 2>&1; echo synccheck rc=$?
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_exchange.py > gpurun_out/r2f_memcheck.log 2>&1; echo memcheck rc=$?
tail -5 gpurun_out/r2f_cfg3.log; tail -3 gpurun_out/r2f_synccheck.log gpurun_out/r2f_memcheck.log; cat gpurun_out/r2f_tf32.log
