"""Per-GEMM accuracy (LSGD_TC_KCHUNK / LSGD_TC_TEST_WS select the variant) of the tcgen05 split-TF32 kernels against float64, beside plain fp32 (torch, TF32 off), on the
cfg3 shapes with cfg3-like operands (non-negative post-ReLU activations, N(0, 1/fan_in) weights)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_tc import tc_gemm, rel  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
rng = np.random.default_rng(0)
B, F, H = 512, 4096, 8192
for name, M, Nn, K, a_mn, b_mn, epi, nonneg in [
    ("fwd L1  [B,H]x[H,H]^T", B, H, H, 0, 0, 0, True),
    ("fwd L0  [B,F]x[H,F]^T", B, H, F, 0, 0, 0, False),
    ("dX  L1  [B,H]x[H,H]", B, H, H, 0, 1, 2, False),
    ("dW  L1  [H,B]x[H,B]", H, H, B, 1, 1, 1, True),
    ("dW  L0  [H,B]x[F,B]", H, F, B, 1, 1, 1, False),
]:
    A = rng.standard_normal((M, K)).astype(np.float32)
    if nonneg:
        A = np.maximum(A, 0)
    Bm = (rng.standard_normal((Nn, K)) / np.sqrt(K)).astype(np.float32)
    ref = A.astype(np.float64) @ Bm.astype(np.float64).T
    tc = tc_gemm(A, Bm, a_mn, b_mn, epi=epi, div=1.0, bias=np.zeros(Nn, np.float32) if epi == 0 else None,
                 mask=np.ones((M, Nn), np.float32) if epi == 2 else None)
    f32 = (torch.tensor(A, device="cuda") @ torch.tensor(Bm, device="cuda").T).cpu().numpy()
    print(f"{name:24s} K={K:5d}  tc {rel(tc, ref):.2e}  fp32 {rel(f32, ref):.2e}  "
          f"max|tc-ref| {np.abs(tc - ref).max():.2e}  mean(tc-ref) {np.mean(tc - ref):+.2e}", flush=True)
