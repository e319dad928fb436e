set -x
for kc in ${KCS:-0 256 512 1024}; do
  for ws in 0 1; do
    echo "== KCHUNK=$kc WS=$ws"
    LSGD_TC_KCHUNK=$kc LSGD_TC_TEST_WS=$ws timeout -s KILL 120 python tools/accuracy_probe.py
    LSGD_TC_KCHUNK=$kc LSGD_TC_TEST_WS=$ws timeout -s KILL 120 python tools/gemm_bench.py 2>&1 | head -8
  done
done
