"""Tensor-core GEMM shape sweep (device-timed) for tuning: the cfg3 step's GEMMs and variants."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_05936_b200 import _native as N
fn = N.lib.lsgd_b200_test_gemm_timed
fn.argtypes = [C.c_int32] * 7 + [C.c_void_p]
shapes = [  # name, a_mn, b_mn, epi, M, N, K
    ("fwd L0", 0, 0, 0, 512, 8192, 4096), ("fwd L1", 0, 0, 0, 512, 8192, 8192), ("fwd L2", 0, 0, 0, 512, 512, 8192),
    ("dX L2", 0, 1, 2, 512, 8192, 512), ("dX L1", 0, 1, 2, 512, 8192, 8192),
    ("dW L2", 1, 1, 1, 512, 8192, 512), ("dW L1", 1, 1, 1, 8192, 8192, 512), ("dW L0", 1, 1, 1, 8192, 4096, 512),
    ("dW L2 as KK", 0, 0, 1, 512, 8192, 512), ("dW L1 as KK", 0, 0, 1, 8192, 8192, 512),
]
tot = 0
for name, a, b, e, M, Nn, K in shapes:
    ms = C.c_double()
    N.check(fn(a, b, e, M, Nn, K, 10, C.byref(ms)))
    tf = 2 * M * Nn * K / (ms.value * 1e-3) / 1e12
    print(f"{name:14s} {M:6d}x{Nn:6d}x{K:6d}  {ms.value*1e3:9.1f} us  {tf:7.1f} TF/s(3xTF32 eff)", flush=True)
