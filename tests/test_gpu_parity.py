"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the reference goldens.

Contract:
  * fp64 parity mode: per-coordinate |a-b|/max(|a|,1e-8) <= 1e-8 over every iterate (the reference's own metric,
    executors.cpp:577) — in practice ~1e-13, the only non-bitwise steps being CUDA's exp/log vs glibc's;
  * fp32 (production) mode: ||w_t - w_t^ref||_2 / ||w_t^ref||_2 <= 1e-5 for every t <= 100, plain and momentum;
  * integer artefacts (indices, shards, topology) bit-exact; replicas bitwise identical; run-to-run bitwise
    reproducible; LSGD G=1 bitwise equal to ordered CSGD (test_executors.cpp:136-145).
"""
import dataclasses
import json
import os

import numpy as np
import pytest

import paper_1906_05936_b200 as lsgd
from paper_1906_05936_b200 import kernels
from paper_1906_05936_b200.executors import compare_histories

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FX = np.load(os.path.join(GOLD, "ref_fixtures.npz"))
META = json.load(open(os.path.join(GOLD, "ref_fixtures.json")))

FP64_TOL = 1e-8   # per-coordinate, the reference's verify tolerance
FP32_TOL = 1e-5   # norm-wise relative, BASELINE north star


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    from paper_1906_05936_b200 import host
    if host.device_count() < 1:
        pytest.fail("no GPU visible: the gpu-marked tests must run on a B200")


def spec_to_cfg(name, **b200):
    s = META["specs"][name]
    keys = ("algorithm", "n_workers", "n_groups", "layer_sizes", "n_samples", "n_features", "n_classes", "spread",
            "mode", "base_lr", "momentum", "weight_decay", "warmup_epochs", "decay_every_epochs", "decay_factor",
            "local_batch", "epochs", "iterations", "seed", "init_scale")
    cfg = lsgd.TrainConfig(**{k: s[k] for k in keys})
    cfg.record_history = True
    for k, v in b200.items():
        setattr(cfg.b200, k, v)
    return cfg


def golden_hist(name):
    return FX[f"{name}_hist"], FX[f"{name}_hist_rows"]


# ------------------------------------------------------------------------------------------ kernel seam
def test_batch_gradient_fp64_matches_reference():
    x, y = lsgd_host_data()
    g, loss = kernels.batch_gradient([32, 16, 10], FX["init_w0"], x, y, FX["sampler_cfg1"][0], dtype="fp64")
    ref = FX["grad_w0_batch0"]
    assert np.max(np.abs(g - ref) / np.maximum(np.abs(ref), 1e-8)) <= 1e-12
    assert abs(loss - FX["loss_w0_batch0"][0]) <= 1e-14
    g, loss = kernels.batch_gradient([8, 12, 7, 5], FX["deep_w"], FX["deep_x"], FX["deep_y"], FX["deep_idx"],
                                     dtype="fp64")
    ref = FX["deep_grad"]
    assert np.max(np.abs(g - ref) / np.maximum(np.abs(ref), 1e-8)) <= 1e-12


def test_batch_gradient_fp32_matches_reference():
    x, y = lsgd_host_data()
    g, loss = kernels.batch_gradient([32, 16, 10], FX["init_w0"], x, y, FX["sampler_cfg1"][0], dtype="fp32")
    ref = FX["grad_w0_batch0"]
    assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= 1e-6
    assert abs(loss - FX["loss_w0_batch0"][0]) <= 1e-6


def test_closed_form_gradient_and_edge_batches():
    g, loss = kernels.batch_gradient([2, 2], np.zeros(6), np.array([[1.0, 2.0]]), np.array([0]), [0])
    assert np.allclose(g, [-0.5, -1.0, 0.5, 1.0, -0.5, 0.5], atol=1e-15) and abs(loss - np.log(2)) < 1e-12
    with pytest.raises(lsgd.LsgdError):  # label out of range (mlp.cpp:136-140)
        kernels.batch_gradient([2, 2], np.zeros(6), np.array([[1.0, 2.0]]), np.array([5]), [0])


def test_collectives_bitwise_in_reference_order():
    c = FX["coll_contrib"]
    assert np.array_equal(kernels.collective("reduce", c, root=2)[2], FX["coll_reduce_root2"])
    out = kernels.collective("allreduce", c)
    for r in range(c.shape[0]):
        assert np.array_equal(out[r], FX["coll_allreduce"])
    b = kernels.collective("broadcast", c, root=1)
    assert all(np.array_equal(b[r], c[1]) for r in range(c.shape[0]))
    assert kernels.collective("reduce", [[1, 2], [3, 4], [5, 6]])[0].tolist() == [9, 12]
    # x2 commutes bitwise (test_transport.cpp:228-246)
    assert np.array_equal(kernels.collective("allreduce", 2 * c)[0], 2 * FX["coll_allreduce"])


def test_sgd_update_bitwise_fp64():
    from oracle import Oracle
    o = Oracle("port")
    rng = np.random.default_rng(0)
    w, d, v = rng.standard_normal(1001), rng.standard_normal(1001), rng.standard_normal(1001)
    for mode in ("plain", "momentum"):
        gw, gv = kernels.sgd_update(w, d, v if mode == "momentum" else None, mode, 0.9, 1e-4, 0.05)
        ow, ov = o.sgd_update(w, d, v if mode == "momentum" else None, mode, 0.9, 1e-4, 0.05)
        assert np.array_equal(gw, ow)
        if mode == "momentum":
            assert np.array_equal(gv, ov)
    gw, _ = kernels.sgd_update([1.0], [0.5], None, "plain", 0.9, 1e-4, 0.1)
    assert abs(gw[0] - 0.95) < 1e-15
    with pytest.raises(lsgd.LsgdError):
        kernels.sgd_update([1.0], [np.inf], None, "plain", 0.9, 1e-4, 0.1)


def lsgd_host_data():
    from paper_1906_05936_b200 import host
    return host.generate_synthetic(42, 5000, 32, 10, 10.0)


# ------------------------------------------------------------------------------------------ training step
FP64_RUNS = ["seq", "lsgd_1x1", "lsgd_2x2", "lsgd_2x4", "lsgd_4x2", "lsgd_1x8", "csgd_4", "lsgd_2x1",
             "lsgd_2x2_mom", "exec_lsgd_4x2"]


@pytest.mark.parametrize("name", FP64_RUNS)
def test_fp64_training_matches_reference_per_coordinate(name):
    cfg = spec_to_cfg(name, dtype="fp64", n_devices=1, global_allreduce="ordered")
    r = lsgd.run_train(cfg)
    ref, rows = golden_hist(name)
    e = compare_histories(ref, r.param_history[rows], name)
    assert e.max_rel_deviation <= FP64_TOL, e
    assert np.allclose(r.loss_history, FX[f"{name}_loss"], rtol=1e-10, atol=1e-14)
    assert np.array_equal(r.lr_history, FX[f"{name}_lr"])
    assert r.gpu_launches > 0


@pytest.mark.parametrize("name", ["lsgd_2x2", "lsgd_1x1", "lsgd_2x2_mom", "lsgd_1x1_mom", "lsgd_2x4_mom", "seq"])
def test_fp32_training_matches_reference_normwise(name):
    cfg = spec_to_cfg(name, dtype="fp32", n_devices=1, global_allreduce="ordered")
    r = lsgd.run_train(cfg)
    ref, rows = golden_hist(name)
    e = compare_histories(ref, r.param_history[rows], name)
    assert e.max_normwise_deviation <= FP32_TOL, e
    assert np.allclose(r.loss_history, FX[f"{name}_loss"], rtol=2e-4, atol=1e-6)


def test_replicas_identical_and_never_stale():
    for alg, G in (("lsgd", 2), ("csgd", 1)):
        cfg = lsgd.TrainConfig(algorithm=alg, n_workers=4, n_groups=G, layer_sizes=[16, 8, 4], n_samples=512,
                               n_features=16, n_classes=4, spread=6.0, mode="plain", local_batch=8, iterations=12)
        cfg.b200.n_devices = 1
        r = lsgd.run_train(cfg)
        for w in range(1, 4):
            assert np.array_equal(r.worker_finals[0].view(np.uint64), r.worker_finals[w].view(np.uint64))
        assert (r.version_at_compute == np.arange(12)[None, :]).all()


@pytest.mark.parametrize("dtype", ["fp32", "fp64"])
def test_single_group_lsgd_is_bitwise_ordered_csgd(dtype):
    a = spec_to_cfg("csgd_4", dtype=dtype, n_devices=1)
    b = spec_to_cfg("lsgd_1x4", dtype=dtype, n_devices=1)
    ra, rb = lsgd.run_train(a), lsgd.run_train(b)
    assert np.array_equal(ra.param_history.view(np.uint64), rb.param_history.view(np.uint64))


def test_run_to_run_bitwise_reproducible():
    cfg = spec_to_cfg("lsgd_2x4_mom", dtype="fp32", n_devices=1, global_allreduce="ordered")
    a, b = lsgd.run_train(cfg), lsgd.run_train(cfg)
    assert np.array_equal(a.param_history.view(np.uint32 if False else np.uint64), b.param_history.view(np.uint64))


def test_verify_equivalence_normwise_fp32():
    base = dict(layer_sizes=[32, 16, 10], mode="plain", iterations=50)
    cfgs = [lsgd.TrainConfig(algorithm="sequential", local_batch=64, **base),
            lsgd.TrainConfig(algorithm="csgd", n_workers=4, local_batch=16, **base),
            lsgd.TrainConfig(algorithm="lsgd", n_workers=4, n_groups=2, local_batch=16, **base)]
    for c in cfgs:
        c.b200.n_devices = 1
        c.b200.global_allreduce = "ordered"
    rep = lsgd.verify_equivalence(cfgs, tolerance=1e-5, metric="normwise")
    assert rep.passed, rep


def test_synthetic_gradient_step_matches_closed_form():
    """cfg4-style step at small P: every worker's gradient is the Rng(1000+r) vector, so after T plain steps
    w_T = w_0 - sum_t lr_t * gbar with gbar the ordered LSGD average."""
    from paper_1906_05936_b200 import host
    P, N_, G_ = 4099, 4, 2
    cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=N_, n_groups=G_, local_batch=1, n_samples=64, mode="plain",
                           iterations=5, layer_sizes=[32, 16, 10])
    cfg.b200.model = "synthetic_gradient"
    cfg.b200.synthetic_params = P
    cfg.b200.n_devices = 1
    cfg.b200.global_allreduce = "ordered"
    cfg.b200.dtype = "fp64"
    r = lsgd.run_train(cfg)
    g = np.zeros((N_, P + 1))
    for i in range(N_):
        s = host.splitmix(1000 + i, P + 1)
        g[i] = 1.0 * (2.0 * ((s >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0)
    per = N_ // G_
    sums = []
    for gi in range(G_):
        acc = g[gi * per].copy()
        for i in range(gi * per + 1, (gi + 1) * per):
            acc += g[i]
        acc = (acc + 0.0) / N_
        sums.append(acc)
    gbar = sums[0] + sums[1]
    s0 = host.splitmix(cfg.seed + 1, P)
    w = 0.05 * (2.0 * ((s0 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0)
    for t in range(5):
        w = w - r.lr_history[t] * gbar[:P]
    assert np.array_equal(r.final_params, w)
    assert np.all(r.loss_history == gbar[P])


# ------------------------------------------------------------------------------------------ multi-GPU
@pytest.mark.multigpu
@pytest.mark.parametrize("name,glob", [("lsgd_2x2", "nccl"), ("lsgd_2x2", "ordered"), ("lsgd_2x1", "nccl"),
                                       ("lsgd_1x4", "ordered")])
def test_multi_gpu_matches_reference(name, glob, n_gpus):
    cfg = spec_to_cfg(name, dtype="fp64", global_allreduce=glob)
    if n_gpus < cfg.n_workers:
        pytest.skip(f"needs {cfg.n_workers} GPUs")
    cfg.b200.n_devices = cfg.n_workers
    r = lsgd.run_train(cfg)
    ref, rows = golden_hist(name)
    e = compare_histories(ref, r.param_history[rows], name)
    assert e.max_rel_deviation <= FP64_TOL, e
    for w in range(1, cfg.n_workers):
        assert np.array_equal(r.worker_finals[0].view(np.uint64), r.worker_finals[w].view(np.uint64))
    cfg.b200.n_devices = 1  # emulated ranks on one GPU give the same bits (G <= 2: NCCL's a+b commutes)
    r1 = lsgd.run_train(cfg)
    assert np.array_equal(r1.final_params.view(np.uint64), r.final_params.view(np.uint64))


@pytest.mark.multigpu
@pytest.mark.parametrize("groups,per_group,dtype,glob", [(4, 1, "fp64", "ordered"), (1, 4, "fp64", "ordered"),
                                                         (2, 2, "fp32", "ordered"), (2, 2, "fp32", "nccl")])
def test_multi_gpu_push_exchange_vs_oracle(groups, per_group, dtype, glob, n_gpus, monkeypatch):
    """One worker per GPU runs the push exchange (scatter -> owner ordered sum -> group-sum push -> ordered global
    sum -> gfull push). fp64: per-coordinate vs the oracle (G = 4 / k = 4 make the summation order observable);
    fp32 on a tensor-core-eligible MLP with row-block buckets: norm-wise."""
    n = groups * per_group
    if n_gpus < n:
        pytest.skip(f"needs {n} GPUs")
    if dtype == "fp32":
        monkeypatch.setenv("LSGD_B200_BUCKET_ELEMS", "20000")
        monkeypatch.setenv("LSGD_B200_GEMM_ELEMS", "70000")  # two exchange buckets per weight-gradient GEMM
        cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=n, n_groups=groups, layer_sizes=[256, 512, 256],
                               n_samples=4096, n_features=256, n_classes=256, spread=6.0, mode="momentum",
                               local_batch=128, iterations=10, record_history=True)
    else:
        cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=n, n_groups=groups, layer_sizes=[16, 24, 8], n_samples=512,
                               n_features=16, n_classes=8, spread=6.0, mode="momentum", local_batch=8, iterations=12,
                               record_history=True)
    cfg.b200.dtype = dtype
    cfg.b200.n_devices = n
    cfg.b200.global_allreduce = glob
    r = lsgd.run_train(cfg)
    from oracle import Oracle, TrainSpec
    spec = TrainSpec(**{k: getattr(cfg, k) for k in TrainSpec.__dataclass_fields__ if hasattr(cfg, k)})
    ref = Oracle("port").run_train(spec, history=True)["history"]
    e = compare_histories(ref, r.param_history, "push")
    assert (e.max_rel_deviation if dtype == "fp64" else e.max_normwise_deviation) <= \
        (FP64_TOL if dtype == "fp64" else FP32_TOL), e
    for w in range(1, n):
        assert np.array_equal(r.worker_finals[0].view(np.uint32), r.worker_finals[w].view(np.uint32))


@pytest.mark.parametrize("dtype,tol", [("fp64", FP64_TOL), ("fp32", FP32_TOL)])
def test_row_block_buckets_keep_parity(dtype, tol, monkeypatch):
    """Large layers are exchanged in row blocks (sub-buckets); force several blocks on a small model and check the
    reference iterates are unchanged (per-coordinate in fp64, norm-wise in fp32)."""
    monkeypatch.setenv("LSGD_B200_BUCKET_ELEMS", "100")
    monkeypatch.setenv("LSGD_B200_GEMM_ELEMS", "400")  # several exchange buckets per weight-gradient GEMM block
    cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=4, n_groups=2, layer_sizes=[16, 64, 32, 4], n_samples=512,
                           n_features=16, n_classes=4, spread=6.0, mode="momentum", local_batch=8, iterations=12,
                           record_history=True)
    cfg.b200.dtype = dtype
    cfg.b200.n_devices = 1
    cfg.b200.global_allreduce = "ordered"
    r = lsgd.run_train(cfg)
    from oracle import Oracle, TrainSpec
    spec = TrainSpec(**{k: getattr(cfg, k) for k in TrainSpec.__dataclass_fields__ if hasattr(cfg, k)})
    ref = Oracle("port").run_train(spec, history=True)["history"]
    e = compare_histories(ref, r.param_history, "blocks")
    assert (e.max_rel_deviation if dtype == "fp64" else e.max_normwise_deviation) <= tol, e


@pytest.mark.parametrize("n_devices", [1, 4])
def test_phase_spans_and_io_overlaps_global_allreduce(n_devices, n_gpus, tmp_path):
    """test_executors.cpp:195-220 on the GPU: with injected io (20 ms) and link (12 ms) delays LSGD's mean block is
    shorter than CSGD's, and worker 0's io of block t+1 overlaps the global allreduce of round t; the delays change
    no bits. The recorded spans feed the reference-schema metrics CSV (metrics.cpp:32-44)."""
    if n_gpus < n_devices:
        pytest.skip(f"needs {n_devices} GPUs")
    res = {}
    for alg, G in (("csgd", 1), ("lsgd", 2)):
        cfg = lsgd.TrainConfig(algorithm=alg, n_workers=4, n_groups=G, layer_sizes=[16, 8, 4], n_samples=512,
                               n_features=16, n_classes=4, spread=6.0, local_batch=8, iterations=8,
                               io_delay_s=0.020, global_link_delay_s=0.012)
        cfg.b200.n_devices = n_devices
        cfg.b200.record_phases = True
        res[alg] = (cfg, lsgd.run_train(cfg))
    if n_devices > 1:  # one worker per GPU: the exchange runs on its own streams, concurrently with the next io
        assert res["lsgd"][1].total_wall_s < res["csgd"][1].total_wall_s
        sp = res["lsgd"][1].phase_spans
        for t in range(7):
            io_next, ar = sp[0, t + 1, 0], sp[:, t, 3]
            assert io_next[1] > io_next[0]
            assert any(a[1] > a[0] and a[0] < io_next[1] and io_next[0] < a[1] for a in ar), (t, io_next, ar)
    cfg, r = res["lsgd"]
    # delay determinism (test_transport.cpp jitter cases): the injected delays move kernels in time, never the bits
    quiet = dataclasses.replace(cfg, io_delay_s=0.0, global_link_delay_s=0.0,
                                b200=dataclasses.replace(cfg.b200, record_phases=False))
    assert np.array_equal(lsgd.run_train(quiet).final_params.view(np.uint64), r.final_params.view(np.uint64))
    path = tmp_path / "metrics.csv"
    lsgd.write_metrics_csv(str(path), "gpu", cfg, r)
    rows = path.read_text().splitlines()
    assert rows[0] == lsgd.K_METRICS_HEADER and len(rows) == 9
    io_s = np.array([float(x.split(",")[8]) for x in rows[1:]])
    assert np.all(io_s > 0.015)  # the injected 20 ms io delay shows up in t_io_s


def test_loss_history_longer_than_the_device_ring():
    """Runs past the 65,536-round device loss ring: history() still returns every iteration's loss (the ring is
    spilled to host memory every 32,768 steps; ADVICE r1 found it silently wrapping)."""
    kw = dict(algorithm="lsgd", n_workers=1, n_groups=1, layer_sizes=[8, 4], n_samples=256, n_features=8,
              n_classes=4, spread=6.0, mode="plain", local_batch=4, seed=3)
    long = lsgd.run_train(lsgd.TrainConfig(iterations=70_000, **kw))
    short = lsgd.run_train(lsgd.TrainConfig(iterations=300, **kw))
    assert long.loss_history.shape == (70_000,) and np.isfinite(long.loss_history).all()
    assert np.array_equal(long.loss_history[:300], short.loss_history)  # same rounds, same bits (deterministic)
    assert not np.array_equal(long.loss_history[65_536:65_836], long.loss_history[:300])  # not wrapped


def test_flag_protocol_check():
    """wait_flags_kernel's round-counter check (the stand-in for compute-sanitizer, which is closed on this pool):
    a flag at the awaited round passes, one a round beyond the allowed lead is reported as a protocol violation
    (code 2 -> TransportError in the engine), one below the target times out (code 1)."""
    import ctypes as C
    from paper_1906_05936_b200 import _native as N
    f = N.lib.lsgd_b200_test_wait_flag
    f.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_int32)]
    f.restype = C.c_int
    code = C.c_int32()
    for value, target, lead, want in [(5, 5, 0, 0), (6, 5, 1, 0), (6, 5, 0, 2), (7, 5, 1, 2), (4, 5, 0, 1)]:
        N.check(f(value, target, lead, C.byref(code)))
        assert code.value == want, (value, target, lead, code.value)
