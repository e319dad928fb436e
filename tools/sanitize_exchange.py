"""Run the 2-GPU push exchange under compute-sanitizer (one process, one host thread per GPU: run_train with
b200.n_devices = 2), small configs: LSGD 2x1 fp32 on the tensor-core path (dW-epilogue scatter, fused global update,
flags) and LSGD 2x1 / CSGD 2 fp64 (SIMT kernels). Generous collective timeout: the tools slow kernels 10-100x.

    compute-sanitizer --tool synccheck python tools/sanitize_exchange.py
    compute-sanitizer --tool memcheck  python tools/sanitize_exchange.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1906_05936_b200 as lsgd  # noqa: E402


def run(algo, groups, dtype, layers, iters):
    d = layers[0]
    cfg = lsgd.TrainConfig(algorithm=algo, n_workers=2, n_groups=groups, layer_sizes=layers, n_samples=1024,
                           n_features=d, n_classes=layers[-1], spread=6.0, mode="momentum",
                           local_batch=128 if dtype == "fp32" else 8, iterations=iters)
    cfg.b200.dtype = dtype
    cfg.b200.n_devices = 2
    cfg.collective_timeout_s = 600.0
    r = lsgd.run_train(cfg)
    print(algo, groups, dtype, layers, "final loss", r.loss_history[-1], "launches", r.gpu_launches, flush=True)


if __name__ == "__main__":
    run("lsgd", 2, "fp32", [256, 512, 256], 3)
    run("lsgd", 2, "fp64", [16, 24, 8], 3)
    run("lsgd", 1, "fp64", [16, 24, 8], 3)
    print("sanitize_exchange ok")
