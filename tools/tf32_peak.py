"""Measured dense TF32 tensor-core peak on this B200 (cuBLAS via torch, TF32 math on), the ceiling the split-TF32
(3 MMAs per product) GEMMs are held against: 3xTF32 ceiling = TF32 peak / 3. Writes profiles/r2_tf32_peak.json.

    python tools/tf32_peak.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def tflops(M, N, K, reps=50, long=False):
    a = torch.randn(M, K, device="cuda", dtype=torch.float32)
    b = torch.randn(K, N, device="cuda", dtype=torch.float32)
    for _ in range(5):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = reps * (20 if long else 1)
    e0.record()
    for _ in range(n):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    return 2.0 * M * N * K * n / (e0.elapsed_time(e1) / 1e3) / 1e12


def main():
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    out = {"device": torch.cuda.get_device_name(0), "method": "torch.matmul fp32 inputs, allow_tf32 (cuBLAS TF32)",
           "shapes": {}}
    for s in [(8192, 8192, 8192), (16384, 16384, 8192), (512, 8192, 8192), (8192, 8192, 512)]:
        out["shapes"]["x".join(map(str, s))] = tflops(*s)
    out["tf32_tflops_burst"] = max(out["shapes"].values())
    out["tf32_tflops_sustained"] = tflops(8192, 8192, 8192, long=True)
    out["split_tf32_ceiling_tflops"] = out["tf32_tflops_sustained"] / 3.0
    torch.backends.cuda.matmul.allow_tf32 = False
    out["fp32_simt_tflops"] = tflops(8192, 8192, 8192, reps=10)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", "r2_tf32_peak.json"), "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
