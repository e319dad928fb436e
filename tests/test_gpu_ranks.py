"""One process per GPU through the rank API (lsgd_b200_rank_create -> export -> connect over a gloo allgather ->
step -> drain), the way bench.py / torchrun drive it (run_rank seam, executors.hpp:143-144): the final parameters
match the oracle (fp64 per coordinate, fp32 tensor-core path norm-wise) and agree bitwise across ranks, and a peer
that never arrives surfaces as TransportError (the collective timeout of transport.cpp / tcp.cpp) instead of a hang.
"""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cfg(dtype, n, groups):
    import paper_1906_05936_b200 as lsgd
    if dtype == "fp64":
        cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=n, n_groups=groups, layer_sizes=[16, 24, 8], n_samples=512,
                               n_features=16, n_classes=8, spread=6.0, mode="momentum", local_batch=8, iterations=12)
    else:  # tensor-core-eligible: the production schedule (buckets, streams, backward order of the layout)
        cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=n, n_groups=groups, layer_sizes=[256, 512, 256],
                               n_samples=4096, n_features=256, n_classes=256, spread=6.0, mode="momentum",
                               local_batch=128, iterations=10)
    cfg.b200.dtype = dtype
    return cfg


def _apply(cfg, over):
    for key, v in (over or {}).items():
        obj = cfg
        *path, last = key.split(".")
        for p in path:
            obj = getattr(obj, p)
        setattr(obj, last, v)
    return cfg


def _worker(rank, world, port, dtype, groups, mode, out, env=None, over=None):
    sys.path.insert(0, ROOT)
    os.environ.update(env or {})  # before the library reads its knobs (first Rank)
    import torch
    import torch.distributed as dist

    import paper_1906_05936_b200 as lsgd
    from paper_1906_05936_b200.executors import Rank

    torch.cuda.set_device(rank)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = _apply(_cfg(dtype, world, groups), over)
        if mode == "timeout":
            cfg.collective_timeout_s = 2.0
        r = Rank(cfg, rank, rank)
        blobs = [None] * world
        dist.all_gather_object(blobs, r.export())
        r.connect(blobs)
        r.synchronize()
        if mode == "train":
            r.step(cfg.iterations)
            r.drain()
            out[rank] = r.params()
        elif rank == 0:  # rank 1 never steps: every flag rank 0 waits for stays unset
            try:
                r.step(1)
                r.synchronize()
                out["err"] = None
            except lsgd.LsgdError as e:
                out["err"] = type(e).__name__
                out["msg"] = str(e)
        dist.barrier()
        r.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _spawn(world, dtype, groups, mode, env=None, over=None):
    import torch.multiprocessing as mp
    mgr = mp.get_context("spawn").Manager()  # no fork() of this multi-threaded process
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), dtype, groups, mode, out, env, over), nprocs=world, join=True)
    return dict(out)


@pytest.mark.parametrize("groups,per_group,dtype", [(2, 1, "fp64"), (2, 2, "fp64"), (1, 2, "fp64"), (2, 2, "fp32")])
def test_process_per_gpu_ranks_match_oracle(groups, per_group, dtype, n_gpus):
    n = groups * per_group
    if n_gpus < n:
        pytest.skip(f"needs {n} GPUs")
    out = _spawn(n, dtype, groups, "train")
    from oracle import Oracle, TrainSpec
    cfg = _cfg(dtype, n, groups)
    spec = TrainSpec(**{k: getattr(cfg, k) for k in TrainSpec.__dataclass_fields__ if hasattr(cfg, k)})
    ref = Oracle("port").run_train(spec)["final_params"]
    w0 = out[0]
    if dtype == "fp64":
        rel = np.abs(w0 - ref) / np.maximum(np.abs(ref), 1e-8)
        assert rel.max() <= 1e-8, rel.max()
    else:
        dev = np.linalg.norm(w0 - ref) / np.linalg.norm(ref)
        assert dev <= 1e-5, dev
    for q in range(1, n):  # every replica holds the same bits
        assert np.array_equal(out[q].view(np.uint64), w0.view(np.uint64))


def test_missing_peer_is_a_transport_error_not_a_hang(n_gpus):
    if n_gpus < 2:
        pytest.skip("needs 2 GPUs")
    out = _spawn(2, "fp64", 2, "timeout")
    assert out["err"] == "TransportError", out


@pytest.mark.parametrize("groups,per_group", [(2, 1), (2, 2)])
def test_hbm_weight_split_is_bitwise_the_smem_split_multi_gpu(groups, per_group, n_gpus):
    """LSGD_TC_WSPLIT=0 (forward / dX GEMMs read the TF32 hi/lo weights the updates write to HBM) gives the same bits
    as the default in-SMEM split at N > 1, where each owner updates its own slot inside the fused global kernel
    (global_update_kernel must refresh w_hi / w_lo of that slot too)."""
    n = groups * per_group
    if n_gpus < n:
        pytest.skip(f"needs {n} GPUs")
    smem = _spawn(n, "fp32", groups, "train")
    hbm = _spawn(n, "fp32", groups, "train", env={"LSGD_TC_WSPLIT": "0"})
    for q in range(n):
        assert np.array_equal(smem[q].view(np.uint64), hbm[q].view(np.uint64)), q


FLAT = {"algorithm": "csgd", "n_groups": 1, "b200.csgd_nccl": True}


@pytest.mark.parametrize("n,dtype", [(2, "fp64"), (4, "fp64"), (2, "fp32"), (4, "fp32")])
def test_flat_nccl_csgd_bucketed_matches_oracle(n, dtype, n_gpus):
    """The flat-allreduce baseline (CSGD, per-bucket ncclAllReduce on the comm stream as each dW block lands, update
    per bucket on the update stream) against the oracle's CSGD (executors.cpp:132-188). N = 2: a + b commutes, so
    NCCL's sum is the reference's; N = 4: NCCL's reduction order differs from the reference's ascending order, so
    fp64 is held per-coordinate to 1e-8 (the reference's verify tolerance), fp32 norm-wise to 1e-5."""
    if n_gpus < n:
        pytest.skip(f"needs {n} GPUs")
    out = _spawn(n, dtype, 1, "train", over=FLAT)
    from oracle import Oracle, TrainSpec
    cfg = _apply(_cfg(dtype, n, 1), FLAT)
    spec = TrainSpec(**{k: getattr(cfg, k) for k in TrainSpec.__dataclass_fields__ if hasattr(cfg, k)})
    assert spec.algorithm == "csgd"
    ref = Oracle("port").run_train(spec)["final_params"]
    w0 = out[0]
    if dtype == "fp64":
        rel = np.abs(w0 - ref) / np.maximum(np.abs(ref), 1e-8)
        assert rel.max() <= 1e-8, rel.max()
    else:
        dev = np.linalg.norm(w0 - ref) / np.linalg.norm(ref)
        assert dev <= 1e-5, dev
    for q in range(1, n):
        assert np.array_equal(out[q].view(np.uint64), w0.view(np.uint64))


@pytest.mark.parametrize("over", [{"b200.global_allreduce": "nccl"}, FLAT], ids=["lsgd_global_nccl", "csgd_flat_nccl"])
def test_missing_peer_on_nccl_is_a_transport_error_not_a_hang(over, n_gpus):
    """A peer that never issues its collective: the NCCL watchdog aborts the communicator after
    collective_timeout_s and the step raises TransportError (inprocess.cpp:44-49), instead of blocking forever."""
    if n_gpus < 2:
        pytest.skip("needs 2 GPUs")
    out = _spawn(2, "fp64", 1 if over is FLAT else 2, "timeout", over=over)
    assert out["err"] == "TransportError", out


def test_caller_dataset_through_upload_dataset(n_gpus):
    """run_rank(cfg, const Dataset&, ...) (executors.hpp:143-144) -> lsgd_b200_rank_upload_dataset: uploading the very
    blobs the rank generated gives bitwise the same training; a different dataset gives different iterates; shape and
    label errors are ConfigErrors (dataset.cpp's checks)."""
    import paper_1906_05936_b200 as lsgd
    from paper_1906_05936_b200 import host
    from paper_1906_05936_b200.executors import Rank

    def train(data=None):
        cfg = _cfg("fp64", 1, 1)
        r = Rank(cfg, 0, 0)
        r.connect([r.export()])
        if data is not None:
            r.upload_dataset(*data)
        r.step(cfg.iterations)
        r.drain()
        w = r.params()
        r.close()
        return w

    cfg = _cfg("fp64", 1, 1)
    x, y = host.generate_synthetic(cfg.seed, cfg.n_samples, cfg.n_features, cfg.n_classes, cfg.spread)
    base = train()
    same = train((x, y))
    assert np.array_equal(base.view(np.uint64), same.view(np.uint64))
    other = train((x[::-1].copy(), y[::-1].copy()))
    assert not np.array_equal(base, other)
    r = Rank(cfg, 0, 0)
    with pytest.raises(lsgd.ConfigError):
        r.upload_dataset(x[:, :-1], y)
    with pytest.raises(lsgd.ConfigError):
        r.upload_dataset(x[:-1], y[:-1])
    bad = y.copy()
    bad[3] = cfg.n_classes
    with pytest.raises(lsgd.ConfigError):
        r.upload_dataset(x, bad)
    r.close()


@pytest.mark.parametrize("groups,per_group,dtype", [(2, 1, "fp32"), (2, 2, "fp32"), (4, 1, "fp64"), (4, 1, "fp32")])
def test_sliced_global_is_bitwise_the_whole_slot_form(groups, per_group, dtype, n_gpus):
    """The global stage sliced over each slot's G owners (reduce-scatter + all-gather; LSGD_B200_SLICED_GLOBAL,
    default for G > 2) computes every element with the same ordered sums as the whole-slot form, so both give the
    same bits on every replica — and fp64 stays per-coordinate on the oracle."""
    n = groups * per_group
    if n_gpus < n:
        pytest.skip(f"needs {n} GPUs")
    on = _spawn(n, dtype, groups, "train", env={"LSGD_B200_SLICED_GLOBAL": "1"})
    off = _spawn(n, dtype, groups, "train", env={"LSGD_B200_SLICED_GLOBAL": "0"})
    for q in range(n):
        assert np.array_equal(on[q].view(np.uint64), off[q].view(np.uint64)), q
        assert np.array_equal(on[q].view(np.uint64), on[0].view(np.uint64)), q
    if dtype == "fp64":
        from oracle import Oracle, TrainSpec
        cfg = _cfg(dtype, n, groups)
        spec = TrainSpec(**{k: getattr(cfg, k) for k in TrainSpec.__dataclass_fields__ if hasattr(cfg, k)})
        ref = Oracle("port").run_train(spec)["final_params"]
        rel = np.abs(on[0] - ref) / np.maximum(np.abs(ref), 1e-8)
        assert rel.max() <= 1e-8, rel.max()


@pytest.mark.parametrize("groups,per_group,dtype", [(2, 2, "fp32"), (4, 1, "fp64"), (1, 4, "fp64"), (2, 1, "fp64")])
def test_push_exchange_is_deterministic_under_jitter(groups, per_group, dtype, n_gpus):
    """Transport conformance on the real NVLink kernels (test_transport.cpp:135-269 jitter cases): every rank
    delays each bucket's exchange by a pseudo-random 0..2000 us (LSGD_B200_JITTER_US), so flags are reached in
    varying orders across GPUs; the iterates are bitwise those of the undelayed run on every replica (and fp64 stays
    per-coordinate on the oracle)."""
    n = groups * per_group
    if n_gpus < n:
        pytest.skip(f"needs {n} GPUs")
    calm = _spawn(n, dtype, groups, "train")
    jit = _spawn(n, dtype, groups, "train", env={"LSGD_B200_JITTER_US": "2000"})
    for q in range(n):
        assert np.array_equal(jit[q].view(np.uint64), calm[q].view(np.uint64)), q


@pytest.mark.parametrize("groups,per_group", [(2, 1), (2, 2)])
def test_backward_order_changes_no_bits(groups, per_group, n_gpus):
    """LSGD_B200_BWD_SEQ reorders the backward's dX / dW GEMMs (and with them the exchange and update order): the
    same kernels on the same data, so every order gives the same bits (256-512-256: x1 = dX_1, w0 / w1 = dW)."""
    n = groups * per_group
    if n_gpus < n:
        pytest.skip(f"needs {n} GPUs")
    a = _spawn(n, "fp32", groups, "train", env={"LSGD_B200_BWD_SEQ": "w1,x1,w0"})
    b = _spawn(n, "fp32", groups, "train", env={"LSGD_B200_BWD_SEQ": "x1,w0,w1"})
    for q in range(n):
        assert np.array_equal(a[q].view(np.uint64), b[q].view(np.uint64)), q


@pytest.mark.parametrize("groups,per_group,dtype", [(2, 2, "fp32"), (1, 4, "fp64"), (1, 2, "fp32")])
def test_pulled_averages_are_bitwise_the_pushed_ones(groups, per_group, dtype, n_gpus):
    """LSGD_B200_PULL_AVG: members read the slot owners' averages over NVLink inside their update instead of having
    them pushed into gfull first — the same values, so the same bits (and fp64 per-coordinate on the oracle)."""
    n = groups * per_group
    if n_gpus < n:
        pytest.skip(f"needs {n} GPUs")
    pull = _spawn(n, dtype, groups, "train", env={"LSGD_B200_PULL_AVG": "1"})
    push = _spawn(n, dtype, groups, "train", env={"LSGD_B200_PULL_AVG": "0"})
    for q in range(n):
        assert np.array_equal(pull[q].view(np.uint64), push[q].view(np.uint64)), q
    if dtype == "fp64":
        from oracle import Oracle, TrainSpec
        cfg = _cfg(dtype, n, groups)
        spec = TrainSpec(**{k: getattr(cfg, k) for k in TrainSpec.__dataclass_fields__ if hasattr(cfg, k)})
        ref = Oracle("port").run_train(spec)["final_params"]
        assert (np.abs(pull[0] - ref) / np.maximum(np.abs(ref), 1e-8)).max() <= 1e-8


@pytest.mark.parametrize("groups,per_group,dtype", [(2, 2, "fp32"), (2, 2, "fp64")])
def test_direct_exchange_is_bitwise_the_three_hop_form(groups, per_group, dtype, n_gpus):
    """LSGD_B200_DIRECT: members copy their sub-slices straight to every group's slot owner, which forms all group sums
    itself (no owner reduce, no group-sum hop) — the same ordered sums, so the same bits; fp64 on the oracle."""
    n = groups * per_group
    if n_gpus < n:
        pytest.skip(f"needs {n} GPUs")
    d = _spawn(n, dtype, groups, "train", env={"LSGD_B200_DIRECT": "1"})
    h = _spawn(n, dtype, groups, "train", env={"LSGD_B200_DIRECT": "0"})
    for q in range(n):
        assert np.array_equal(d[q].view(np.uint64), h[q].view(np.uint64)), q
    if dtype == "fp64":
        from oracle import Oracle, TrainSpec
        cfg = _cfg(dtype, n, groups)
        spec = TrainSpec(**{k: getattr(cfg, k) for k in TrainSpec.__dataclass_fields__ if hasattr(cfg, k)})
        ref = Oracle("port").run_train(spec)["final_params"]
        assert (np.abs(d[0] - ref) / np.maximum(np.abs(ref), 1e-8)).max() <= 1e-8


@pytest.mark.parametrize("groups,per_group,dtype", [(1, 4, "fp32"), (1, 4, "fp64"), (2, 2, "fp32"), (1, 2, "fp64")])
def test_nvls_multicast_fanout_is_bitwise_the_unicast_push(groups, per_group, dtype, n_gpus):
    """LSGD_B200_NVLS: the slot owner stores each averaged vector once into an NVSwitch multicast object bound to
    its group's gfull buffers (multimem.st) instead of k-1 unicast NVLink stores — a copy, so the same bits; fp64
    also per-coordinate on the oracle. One process per GPU (the object is shared as a file descriptor)."""
    n = groups * per_group
    if n_gpus < n:
        pytest.skip(f"needs {n} GPUs")
    mc = _spawn(n, dtype, groups, "train", env={"LSGD_B200_NVLS": "1"})
    uc = _spawn(n, dtype, groups, "train", env={"LSGD_B200_NVLS": "0"})
    for q in range(n):
        assert np.array_equal(mc[q].view(np.uint64), uc[q].view(np.uint64)), q
    if dtype == "fp64":
        from oracle import Oracle, TrainSpec
        cfg = _cfg(dtype, n, groups)
        spec = TrainSpec(**{k: getattr(cfg, k) for k in TrainSpec.__dataclass_fields__ if hasattr(cfg, k)})
        ref = Oracle("port").run_train(spec)["final_params"]
        assert (np.abs(mc[0] - ref) / np.maximum(np.abs(ref), 1e-8)).max() <= 1e-8


def test_nvls_in_the_threaded_world(n_gpus):
    """The same multicast fan-out in the one-process world (run_train, one host thread per GPU): 1x4 fp64 on the
    oracle per coordinate."""
    if n_gpus < 4:
        pytest.skip("needs 4 GPUs")
    import subprocess
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from test_gpu_ranks import _cfg\n"
        "import paper_1906_05936_b200 as lsgd\n"
        "from oracle import Oracle, TrainSpec\n"
        "cfg = _cfg('fp64', 4, 1); cfg.b200.n_devices = 4\n"
        "w = lsgd.run_train(cfg).final_params\n"
        "spec = TrainSpec(**{k: getattr(cfg, k) for k in TrainSpec.__dataclass_fields__ if hasattr(cfg, k)})\n"
        "ref = Oracle('port').run_train(spec)['final_params']\n"
        "print((np.abs(w - ref) / np.maximum(np.abs(ref), 1e-8)).max())\n" % (ROOT, os.path.join(ROOT, "tests")))
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LSGD_B200_NVLS="1"), cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= 1e-8
