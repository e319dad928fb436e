"""Per-bucket chain of the push exchange on every rank (gpurun_out/timeline_rank<r>.txt from tools/timeline.py
--all-ranks): scatter / wait / reduce / global / update spans of one step, relative to its first forward GEMM."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rows = {}
for r in range(n):
    L = [l.split() for l in open(os.path.join(ROOT, "gpurun_out", f"timeline_rank{r}.txt"))]
    starts = [float(l[2]) for l in L if l[0] == "gemm" and l[1] == "100"]
    t0, t1 = starts[1], starts[2]
    rows[r] = [(l[0], l[1], float(l[2]) - t0, float(l[3]) - t0) for l in L if t0 - 0.001 <= float(l[2]) < t1]
    print("rank", r, "step", round(t1 - t0, 3), "ms")
fams = ["scatter", "wait", "reduce", "global", "update"]
buckets = sorted({t for r in rows for f, t, a, e in rows[r] if f in fams}, key=int)
for b in buckets:
    print("bucket", b)
    for r in range(n):
        print("  r%d" % r, "  ".join(f"{f[:3]} {a:.3f}-{e:.3f}" for f, t, a, e in rows[r] if t == b and f in fams))
