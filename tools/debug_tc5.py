import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1906_05936_b200 import _native as N, host
from paper_1906_05936_b200.executors import init_params
fn = N.lib.lsgd_b200_test_tc_step
fn.argtypes = [C.c_int32, C.c_void_p, C.c_int32] + [C.c_void_p] * 7
L = [256, 512, 256]; B = 128
x, y = host.generate_synthetic(42, 2048, 256, 256, 10.0)
w = init_params(L, 43, 0.05).astype(np.float32)
idx = np.arange(B) * 5
xb = np.ascontiguousarray(x[idx].astype(np.float32)); yb = np.ascontiguousarray(y[idx].astype(np.int32))
Ls = (C.c_int32 * 3)(*L)
P = w.size
def run():
    act = np.zeros(B * (512 + 256), np.float32); dl = np.zeros(B * 256, np.float32); g = np.zeros(P, np.float32); l = np.zeros(1, np.float32)
    N.check(fn(3, Ls, B, w.ctypes.data, xb.ctypes.data, yb.ctypes.data, act.ctypes.data, dl.ctypes.data, g.ctypes.data, l.ctypes.data))
    return act, dl, g, l
W0 = w[:256*512].reshape(512, 256).astype(np.float64); b0 = w[256*512:256*512+512].astype(np.float64)
o1 = 256*512+512
W1 = w[o1:o1+512*256].reshape(256, 512).astype(np.float64); b1 = w[o1+512*256:].astype(np.float64)
a0 = np.maximum(xb.astype(np.float64) @ W0.T + b0, 0); z = a0 @ W1.T + b1
res = [run() for _ in range(3)]
for i, (act, dl, g, l) in enumerate(res):
    A0 = act[:B*512].reshape(B, 512); Z = act[B*512:].reshape(B, 256)
    print(i, "act0", np.linalg.norm(A0 - a0) / np.linalg.norm(a0), "logits", np.linalg.norm(Z - z) / np.linalg.norm(z), "loss", l,
          "grad vs call0", np.linalg.norm(g - res[0][2]) / np.linalg.norm(res[0][2]), flush=True)
    bad = np.argwhere(np.abs(A0 - a0) > 1e-3 * np.abs(a0).max())
    if len(bad): print("   act0 bad rows", np.unique(bad[:, 0])[:20], "cols", np.unique(bad[:, 1])[:40], len(bad))
    badz = np.argwhere(np.abs(Z - z) > 1e-3 * np.abs(z).max())
    if len(badz): print("   logits bad rows", np.unique(badz[:, 0])[:20], "cols", np.unique(badz[:, 1])[:40], len(badz))
