"""Tensor-core (tcgen05 split-TF32) path: GEMM conformance against float64 products, and the fp32 training step
on a tc-eligible MLP against the fp64 oracle (norm-wise 1e-5, the same contract as the SIMT path)."""
import ctypes as C
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import paper_1906_05936_b200 as lsgd
from paper_1906_05936_b200 import _native as N

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_fn = N.lib.lsgd_b200_test_gemm
_fn.argtypes = [C.c_int32] * 6 + [C.c_void_p] * 4 + [C.c_float, C.c_int32, C.c_void_p]
_fn.restype = C.c_int


def tc_gemm(A, B, a_mn, b_mn, epi=1, bias=None, mask=None, div=1.0, relu=0):
    """A [M,K], B [N,K] logical; stored per major."""
    M, K = A.shape
    Nn = B.shape[0]
    As = np.ascontiguousarray((A.T if a_mn else A).astype(np.float32))
    Bs = np.ascontiguousarray((B.T if b_mn else B).astype(np.float32))
    out = np.zeros((M, Nn), dtype=np.float32)
    bias = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    mask = None if mask is None else np.ascontiguousarray(mask, dtype=np.float32)
    N.check(_fn(a_mn, b_mn, epi, M, Nn, K, As.ctypes.data, Bs.ctypes.data,
                bias.ctypes.data if bias is not None else None, mask.ctypes.data if mask is not None else None,
                div, relu, out.ctypes.data))
    return out


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
def test_gemm_majors_fp32_accurate(a_mn, b_mn):
    rng = np.random.default_rng(1 + 2 * a_mn + b_mn)
    M, Nn, K = 256, 512, 320
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((Nn, K)).astype(np.float32)
    got = tc_gemm(A, B, a_mn, b_mn, epi=1, div=1.0)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    assert rel(got, ref) < 3e-6, rel(got, ref)
    # plain TF32 would be ~1e-3: make sure the split terms are really there
    assert np.abs(got - ref).max() < 1e-3


@pytest.mark.parametrize("M", [128, 384, 768])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 1), (0, 1)])
def test_gemm_single_cta_and_pair_tiles(M, a_mn, b_mn):
    """M % 256 != 0 runs single-CTA 128-row tiles; M = 768 runs CTA-pair (cta_group::2) 256-row tiles."""
    rng = np.random.default_rng(M + 3 * a_mn + b_mn)
    Nn, K = 768, 272
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((Nn, K)).astype(np.float32)
    mask = (rng.standard_normal((M, Nn)) > 0).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    got = tc_gemm(A, B, a_mn, b_mn, epi=1, div=1.0)
    assert rel(got, ref) < 3e-6, rel(got, ref)
    ig = tc_gemm(A, B, a_mn, b_mn, epi=2, mask=mask)
    assert rel(ig, ref * mask) < 3e-6


def test_gemm_epilogues_and_split_k():
    rng = np.random.default_rng(7)
    M, Nn, K = 256, 256, 4096  # few tiles, long K -> split-K with ordered partial reduction
    A = rng.standard_normal((M, K)).astype(np.float32) * 0.1
    B = rng.standard_normal((Nn, K)).astype(np.float32) * 0.1
    bias = rng.standard_normal(Nn).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    fwd = tc_gemm(A, B, 0, 0, epi=0, bias=bias, relu=1)
    assert rel(fwd, np.maximum(ref + bias, 0)) < 3e-6
    wg = tc_gemm(A, B, 1, 1, epi=1, div=512.0)
    assert rel(wg, ref / 512.0) < 3e-6
    mask = (rng.standard_normal((M, Nn)) > 0).astype(np.float32)
    ig = tc_gemm(A, B, 0, 1, epi=2, mask=mask)
    assert rel(ig, ref * mask) < 3e-6
    again = tc_gemm(A, B, 0, 1, epi=2, mask=mask)
    assert np.array_equal(ig.view(np.uint32), again.view(np.uint32))  # deterministic


def tc_cfg(**kw):
    base = dict(algorithm="lsgd", n_workers=2, n_groups=1, layer_sizes=[256, 512, 256], n_samples=2048,
                n_features=256, n_classes=256, spread=10.0, local_batch=128, iterations=30, mode="momentum",
                record_history=True)
    base.update(kw)
    c = lsgd.TrainConfig(**base)
    c.b200.n_devices = 1
    c.b200.global_allreduce = "ordered"
    return c


@pytest.mark.parametrize("mode", ["plain", "momentum"])
def test_tc_training_matches_oracle_normwise(mode):
    from oracle import Oracle, TrainSpec

    cfg = tc_cfg(mode=mode)
    cfg.b200.gemm = "tcgen05"
    r = lsgd.run_train(cfg)
    spec = TrainSpec(**{k: getattr(cfg, k) for k in TrainSpec.__dataclass_fields__})
    ref = Oracle("port").run_train(spec, history=True)["history"]
    dev = np.linalg.norm(r.param_history - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert dev.max() <= 1e-5, dev.max()
    simt = tc_cfg(mode=mode)
    simt.b200.gemm = "simt"
    rs = lsgd.run_train(simt)
    # both fp32 paths sit within 1e-5 of the fp64 oracle; against each other the bound is the sum
    assert np.linalg.norm(rs.final_params - r.final_params) / np.linalg.norm(rs.final_params) <= 2e-5
    for w in range(1, cfg.n_workers):
        assert np.array_equal(r.worker_finals[0].view(np.uint64), r.worker_finals[w].view(np.uint64))


@pytest.mark.parametrize("mode", ["plain", "momentum"])
def test_single_worker_fused_update_is_bitwise_the_update_pass(mode):
    """One worker (N = 1): with LSGD_B200_FUSED_UPDATE the update runs inside the dW / bias epilogues. It must give
    bitwise the iterates of the separate update kernel (the default) and stay within 1e-5 of the oracle."""
    from oracle import Oracle, TrainSpec

    cfg = tc_cfg(mode=mode, n_workers=1, iterations=12)
    cfg.b200.gemm = "tcgen05"
    sep = lsgd.run_train(cfg)
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_1906_05936_b200 as lsgd\n"
        "c = lsgd.TrainConfig(algorithm='lsgd', n_workers=1, n_groups=1, layer_sizes=[256, 512, 256],\n"
        "    n_samples=2048, n_features=256, n_classes=256, spread=10.0, local_batch=128, iterations=12,\n"
        "    mode=%r, record_history=True)\n"
        "c.b200.n_devices = 1; c.b200.global_allreduce = 'ordered'; c.b200.gemm = 'tcgen05'\n"
        "np.save(sys.argv[1], lsgd.run_train(c).param_history)\n" % (ROOT, mode))
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "h.npy")
        env = dict(os.environ, LSGD_B200_FUSED_UPDATE="1")
        subprocess.run([sys.executable, "-c", code, out], check=True, env=env, cwd=ROOT)
        fused = np.load(out)
    assert np.array_equal(fused.view(np.uint64), sep.param_history.view(np.uint64))
    spec = TrainSpec(**{k: getattr(cfg, k) for k in TrainSpec.__dataclass_fields__ if hasattr(cfg, k)})
    ref = Oracle("port").run_train(spec, history=True)["history"]
    dev = np.linalg.norm(fused - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert dev.max() <= 1e-5, dev.max()


def test_weight_split_in_shared_memory_is_bitwise_the_hbm_split():
    """The forward / dX GEMMs split the fp32 weights into TF32 hi/lo in shared memory (default) — the same values the
    separate split pass wrote to HBM (LSGD_TC_WSPLIT=0 path), so the iterates are bitwise identical."""
    cfg = tc_cfg(mode="momentum", n_workers=1, iterations=6)
    cfg.b200.gemm = "tcgen05"
    ws = lsgd.run_train(cfg).param_history
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_1906_05936_b200 as lsgd\n"
        "c = lsgd.TrainConfig(algorithm='lsgd', n_workers=1, n_groups=1, layer_sizes=[256, 512, 256],\n"
        "    n_samples=2048, n_features=256, n_classes=256, spread=10.0, local_batch=128, iterations=6,\n"
        "    mode='momentum', record_history=True)\n"
        "c.b200.n_devices = 1; c.b200.gemm = 'tcgen05'\n"
        "np.save(sys.argv[1], lsgd.run_train(c).param_history)\n" % ROOT)
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "h.npy")
        env = dict(os.environ, LSGD_TC_WSPLIT="0")
        subprocess.run([sys.executable, "-c", code, out], check=True, env=env, cwd=ROOT)
        hbm = np.load(out)
    assert np.array_equal(ws.view(np.uint64), hbm.view(np.uint64))


_KCHUNK_PROBE = """
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
from test_gpu_tc import tc_gemm
rng = np.random.default_rng(11)
M, N, K = 1024, 4096, 4096  # 4 x 16 = 64 pair tiles over 64 slots, and split-free long K: 8 chunks of 512
A = np.maximum(rng.standard_normal((M, K)), 0).astype(np.float32)  # post-ReLU activations: no sign cancellation
B = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
ref = A.astype(np.float64) @ B.astype(np.float64).T
fwd = tc_gemm(A, B, 0, 0, epi=0, bias=np.zeros(N, np.float32))
ig = tc_gemm(A, B, 0, 1, epi=2, mask=np.ones((M, N), np.float32))
M2 = 4096  # 16 x 16 = 256 pair tiles: 4 per CTA pair, so chunk folds and tile epilogues interleave
A2 = np.maximum(rng.standard_normal((M2, K)), 0).astype(np.float32)
ref2 = A2.astype(np.float64) @ B.astype(np.float64).T
fwd2 = tc_gemm(A2, B, 0, 0, epi=0, bias=np.zeros(N, np.float32))
r = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
np.save(sys.argv[1], np.array([r(fwd, ref), r(ig, ref), r(fwd2, ref2)]))
"""


@pytest.mark.parametrize("ws", ["0", "1"])
def test_k_chunked_accumulation_is_fp32_class(ws):
    """The tensor pipe's fp32 accumulation does not round to nearest: one accumulator over K = 4096 drifts ~1.4e-5
    norm-wise from float64. With 512-wide K chunks folded in TMEM (default) the error stays at the one-chunk level
    (~3.6e-6) on one-tile-per-CTA and several-tiles-per-CTA shapes, for the forward and dX forms, with the weights
    split in shared memory (WS=1, the transform interleaved with the folds) or read pre-split from HBM."""
    errs = {}
    for kc in ("512", "0"):
        with tempfile.TemporaryDirectory() as td:
            out = os.path.join(td, "e.npy")
            env = dict(os.environ, LSGD_TC_KCHUNK=kc, LSGD_TC_TEST_WS=ws)
            subprocess.run([sys.executable, "-c", _KCHUNK_PROBE % (ROOT, os.path.join(ROOT, "tests")), out],
                           check=True, env=env, cwd=ROOT)
            errs[kc] = np.load(out)
    assert errs["512"].max() < 6e-6, errs
    assert (errs["0"] > 2.5 * errs["512"]).all(), errs


def test_full_size_cfg3_steps_match_torch_fp64():
    """BASELINE cfg3 at full size (MLP 4096-8192-8192-512, 105M parameters, B_loc = 512, momentum): three steps of
    the production fp32 path (tcgen05 split-TF32 GEMMs, in-SMEM weight split, fused head, eager bucket updates) and of
    the plain-fp32 SIMT path against the same steps restated in float64 with torch on the GPU (autograd MLP, ReLU
    hidden layers, mean softmax-CE of mlp.cpp:60-273, momentum + weight decay of optimizer.cpp:24-42), from the
    oracle's initial weights (rounded to fp32, as the fp32 paths start) and the host sampler's indices / LR.
    At this width any fp32 arithmetic drifts from float64 by ~1e-5 of ||w|| per step (K = 8192 cancellation, ReLU
    masks flipping on near-zero activations) and the dynamics amplify it ~3x per step, so the 1e-5 contract is checked
    at the reference configs (test_tc_training_matches_oracle_normwise). Measured on B200
    (profiles/r1_fullsize_fp64.log): plain fp32 8.3e-6, 2.6e-5, 7.8e-5 after steps 1-3; the tensor-core path with its
    K-chunked accumulation 1.07-1.4x that (3.4x with one accumulator over the whole K, whose tensor-pipe fp32
    accumulation does not round to nearest). Asserted: both below 1e-3, the tensor-core path within 1.6x of plain
    fp32."""
    import torch
    from oracle import Oracle
    from paper_1906_05936_b200 import host

    layers = [4096, 8192, 8192, 512]
    T = 3
    hists = {}
    for gemm in ("tcgen05", "simt"):
        cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=1, n_groups=1, layer_sizes=layers, n_samples=4096,
                               n_features=4096, n_classes=512, spread=10.0, mode="momentum", local_batch=512,
                               iterations=T, record_history=True)
        cfg.b200.n_devices = 1
        cfg.b200.gemm = gemm
        hists[gemm] = lsgd.run_train(cfg).param_history
    w0 = Oracle("port").init_params(layers, cfg.seed + 1, cfg.init_scale).astype(np.float32).astype(np.float64)
    for h in hists.values():
        assert np.array_equal(h[0], w0)
    x, y = host.generate_synthetic(cfg.seed, cfg.n_samples, 4096, 512, cfg.spread)
    idx = host.minibatch_indices(cfg, 0, T)
    dev = torch.device("cuda:0")
    params, off = [], 0
    for k in range(3):
        i, o = layers[k], layers[k + 1]
        params.append(torch.tensor(w0[off:off + i * o].reshape(o, i), dtype=torch.float64, device=dev))
        off += i * o
        params.append(torch.tensor(w0[off:off + o], dtype=torch.float64, device=dev))
        off += o
    vel = [torch.zeros_like(p) for p in params]
    X = torch.tensor(x, dtype=torch.float64, device=dev)
    Y = torch.tensor(y.astype(np.int64), device=dev)
    for t in range(T):
        for p in params:
            p.requires_grad_(True)
        rows = torch.tensor(idx[t].astype(np.int64), device=dev)
        h = X[rows]
        for k in range(3):
            h = h @ params[2 * k].T + params[2 * k + 1]
            if k < 2:
                h = torch.relu(h)
        loss = torch.nn.functional.cross_entropy(h, Y[rows])
        grads = torch.autograd.grad(loss, params)
        lr = host.learning_rate(cfg, t)
        with torch.no_grad():
            for j, (p, g) in enumerate(zip(params, grads)):
                p.requires_grad_(False)
                vel[j] = cfg.momentum * vel[j] + (g + cfg.weight_decay * p)
                p -= lr * vel[j]
        ref = torch.cat([p.reshape(-1) for p in params]).cpu().numpy()
        devs = {g: np.linalg.norm(h_[t + 1] - ref) / np.linalg.norm(ref) for g, h_ in hists.items()}
        print(f"cfg3 step {t}: norm-wise deviation from float64 {devs}", flush=True)
        assert devs["tcgen05"] <= 1e-3 and devs["simt"] <= 1e-3, (t, devs)
        assert devs["tcgen05"] <= 1.6 * max(devs["simt"], 1e-6), (t, devs)


def test_cfg3_steps_match_reference_fixtures():
    """The bench configuration (BASELINE cfg3: MLP 4096-8192-8192-512, 105M parameters, 65,536 blobs, B_loc = 512,
    momentum, one worker) on the production fp32 path, against the UNMODIFIED reference's own run_train in fp64
    (tests/golden/cfg3_ref.npz from tests/golden/make_cfg3_golden.py; executors.cpp:481-521, mlp.cpp:238-273):
      * w_0 is the reference's init rounded to fp32, bit for bit, at every sampled coordinate;
      * after each of the T = 2 steps: ||w_t - w_t^ref|| / ||w_t^ref|| over 66,048 sampled coordinates (16,384 per
        weight matrix + every bias) <= 3e-5 (t = 1) and <= 8e-5 (t = 2), the global and per-weight-matrix norms of
        w_t within the same relative bounds (bias-vector norms within 2e-4), and the accumulated update w_t - w_0
        within 2e-3 of the reference's (relative). Measured on B200: 1.29e-5 / 5.5e-5 sampled, 1.3e-9 / 8.9e-8 on
        ||w_t||, update 6.8e-4 at t = 2 (profiles/r2_acceptance_and_cfg3_vs_reference.log);
      * the per-iteration losses within 3e-5 relative (measured 8.8e-6 at w_0 — fp32 rounding of the initial weights
        and fp32 forward arithmetic — and 1.2e-5 at w_1).
    Why not 1e-5 on w after 100 steps here: at this width fp32 arithmetic itself drifts from float64 by ~1e-5 of
    ||w|| per step and the dynamics amplify it (plain fp32 SIMT: 8.3e-6, 2.6e-5, 7.8e-5 after steps 1-3,
    profiles/r1_fullsize_fp64.log); the 1e-5-after-100-steps contract holds at the reference's configs
    (test_tc_training_matches_oracle_normwise, tests/test_gpu_parity.py)."""
    ref = np.load(os.path.join(ROOT, "tests", "golden", "cfg3_ref.npz"))
    T = int(ref["steps"])
    layers = [4096, 8192, 8192, 512]
    cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=1, n_groups=1, layer_sizes=layers, n_samples=65536,
                           n_features=4096, n_classes=512, spread=10.0, mode="momentum", local_batch=512,
                           iterations=T, record_history=True, seed=42)
    cfg.b200.n_devices = 1
    cfg.b200.gemm = "tcgen05"
    r = lsgd.run_train(cfg)
    h = r.param_history
    idx = ref["idx"]
    assert np.array_equal(h[0][idx], ref["w0"].astype(np.float32).astype(np.float64))
    bounds = {1: 3e-5, 2: 8e-5}
    offs, off = [], 0
    for k in range(3):
        nw = layers[k] * layers[k + 1]
        offs.append((off, off + nw, off + nw, off + nw + layers[k + 1]))
        off += nw + layers[k + 1]
    report = {}
    for t in range(1, T + 1):
        w, wr = h[t][idx], ref[f"w{t}"]
        dev = np.linalg.norm(w - wr) / np.linalg.norm(wr)
        dnorm = abs(np.linalg.norm(h[t]) - float(ref[f"norm{t}"])) / float(ref[f"norm{t}"])
        lnorm = np.array([[np.linalg.norm(h[t][a:b]), np.linalg.norm(h[t][c:d])] for a, b, c, d in offs])
        ldev = np.abs(lnorm - ref[f"lnorm{t}"]) / ref[f"lnorm{t}"]
        upd = np.linalg.norm((w - h[0][idx]) - (wr - ref["w0"])) / np.linalg.norm(wr - ref["w0"])
        report[t] = (dev, dnorm, ldev.max(), upd)
        assert dev <= bounds[t], report
        # weight matrices' norms within the w bound; the bias vectors (8192, 8192, 512 values of ~1e-2) carry the
        # deltas' deviation undiluted: 1e-4 relative (measured 5.9e-5 .. 8.7e-5 at t = 1, 2)
        assert dnorm <= bounds[t] and ldev[:, 0].max() <= bounds[t] and ldev[:, 1].max() <= 2e-4, report
        assert upd <= 2e-3, report
    lrel = np.abs(r.loss_history - ref["loss"]) / np.abs(ref["loss"])
    assert lrel.max() <= 3e-5, (lrel, report)
    print("cfg3 vs reference (sampled dev, norm dev, layer-norm dev, update dev):", report, "loss", lrel)
