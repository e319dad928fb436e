import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1906_05936_b200 import kernels, host
from paper_1906_05936_b200.executors import init_params
from oracle import Oracle
L = [256, 512, 256]
x, y = host.generate_synthetic(42, 2048, 256, 256, 10.0)
w0 = init_params(L, 43, 0.05)
idx = np.arange(128, dtype=np.int32) * 5
g_ref, _ = Oracle("port").batch_gradient(L, w0, x, y, idx)
out = []
for i in range(4):
    g, _ = kernels.batch_gradient(L, w0, x, y, idx, dtype="fp32", gemm="tcgen05")
    out.append(float(np.linalg.norm(g - g_ref) / np.linalg.norm(g_ref)))
print(os.environ.get("LSGD_TC_NOPREFETCH"), os.environ.get("LSGD_TC_NOFREE"), out, flush=True)
