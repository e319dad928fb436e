"""One tensor-core GEMM shape, device-timed (for ncu captures): gemm_one.py a_mn b_mn epi M N K [reps]."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_05936_b200 import _native as N  # noqa: E402

fn = N.lib.lsgd_b200_test_gemm_timed
fn.argtypes = [C.c_int32] * 7 + [C.c_void_p]
a, b, e, M, Nn, K = (int(x) for x in sys.argv[1:7])
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
ms = C.c_double()
N.check(fn(a, b, e, M, Nn, K, reps, C.byref(ms)))
print(f"{M}x{Nn}x{K} a_mn={a} b_mn={b} epi={e}: {ms.value * 1e3:.1f} us  {2 * M * Nn * K / (ms.value * 1e-3) / 1e12:.1f} TF/s")
