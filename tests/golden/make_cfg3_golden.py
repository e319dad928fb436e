"""Reference fixtures for the bench configuration (BASELINE cfg3), from the UNMODIFIED reference library.

Run in the build container (needs /root/reference; builds oracle/_ref/liblsgd_ref.so; ~10-20 min on 8 cores,
~30 GB RAM: the reference's batch_gradient keeps min(32, B) x P per-sample gradients, mlp.cpp:243-245):

    OMP_NUM_THREADS=8 python tests/golden/make_cfg3_golden.py

Runs the reference's own ``run_train`` (proj/src/executors.cpp:481-521) on the wide MLP 4096-8192-8192-512
(P = 104,874,496), ``generate_synthetic(42, 65536, 4096, 512, 10.0)``, momentum SGD, B_loc = 512 on one worker
(sequential = LSGD 1x1, the bench's N=1 layout), T iterations in fp64, and writes ``cfg3_ref.npz``:

  * ``idx``         - seeded sample of parameter coordinates: 16,384 from each weight matrix + every bias;
  * ``w{t}``        - the reference's w_t at those coordinates, t = 0..T;
  * ``norm{t}``     - ||w_t||_2 over all P parameters, and per-layer ``lnorm{t}`` (W_k and b_k of each layer);
  * ``dnorm{t}``    - ||w_t - w_0||_2 (the size of the accumulated update);
  * ``loss``, ``lr`` - the reference's per-iteration loss / learning rate.

The GPU test (tests/test_gpu_tc.py::test_cfg3_steps_match_reference_fixtures) runs the tensor-core fp32 path on the
same config and compares against these.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Oracle, TrainSpec, build  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg3_ref.npz")
LAYERS = [4096, 8192, 8192, 512]
T = int(os.environ.get("CFG3_STEPS", "2"))
PER_MATRIX = 16384


def spec(iterations: int = T) -> TrainSpec:
    # algorithm "sequential": the reference's LSGD 1x1 is bitwise the sequential run (ref_fixtures.json hashes
    # seq = lsgd_1x1), and the sequential executor has no transport whose 30 s receive timeout a minutes-long
    # cfg3 gradient would trip
    return TrainSpec(algorithm="sequential", n_workers=1, n_groups=1, layer_sizes=LAYERS, n_samples=65536,
                     n_features=LAYERS[0], n_classes=LAYERS[-1], spread=10.0, mode="momentum",
                     local_batch=512, iterations=iterations, seed=42)


def layer_ranges(layers):
    """[(w_begin, w_end, b_begin, b_end)] per layer in the reference's flat layout (mlp.cpp:154-166: W_k row-major
    [out, in] then b_k)."""
    out, off = [], 0
    for k in range(len(layers) - 1):
        nw = layers[k] * layers[k + 1]
        out.append((off, off + nw, off + nw, off + nw + layers[k + 1]))
        off += nw + layers[k + 1]
    return out


def sample_indices(layers, seed: int = 7) -> np.ndarray:
    rng = np.random.default_rng(seed)
    idx = []
    for wb, we, bb, be in layer_ranges(layers):
        idx.append(np.sort(rng.choice(np.arange(wb, we), PER_MATRIX, replace=False)))
        idx.append(np.arange(bb, be))
    return np.concatenate(idx).astype(np.int64)


def main():
    build()
    s = spec()
    t0 = time.time()
    out = Oracle("reference").run_train(s, history=True)
    print(f"reference run_train cfg3 T={T}: {time.time() - t0:.0f} s", flush=True)
    h = out["history"]
    idx = sample_indices(LAYERS)
    res = {"idx": idx, "loss": out["loss"], "lr": out["lr"], "steps": np.int64(T)}
    for t in range(T + 1):
        res[f"w{t}"] = h[t, idx]
        res[f"norm{t}"] = np.linalg.norm(h[t])
        res[f"dnorm{t}"] = np.linalg.norm(h[t] - h[0])
        res[f"lnorm{t}"] = np.array([[np.linalg.norm(h[t, wb:we]), np.linalg.norm(h[t, bb:be])]
                                     for wb, we, bb, be in layer_ranges(LAYERS)])
    np.savez_compressed(OUT, **res)
    print("wrote", OUT, {k: (v if np.ndim(v) == 0 else np.shape(v)) for k, v in res.items()})


if __name__ == "__main__":
    main()
