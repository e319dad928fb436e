"""Host-side mirror of the reference executor seam (include/lsgd/executors.hpp) over the C-ABI.

``run_train`` has the reference's signature and result shape (executors.hpp:106-138, executors.cpp:481-521) but
executes on B200s through ``lsgd_b200_run_train``; ``verify_equivalence`` is executors.cpp:523-588 with an added
norm-wise tolerance mode (fp32 parity is defined norm-wise). ``Rank`` wraps the run_rank seam
(executors.hpp:143-144) for one-process-per-GPU worlds.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N

ALGORITHMS = {"sequential": N.SEQUENTIAL, "csgd": N.CSGD, "lsgd": N.LSGD}
PHASES = ("io", "compute", "local_reduce", "global_allreduce", "broadcast", "update")  # executors.hpp:248


@dataclass
class B200Options:
    """The ``b200`` block of a run config (the new ``transport.backend = "b200"``)."""

    dtype: str = "fp32"              # fp32 | fp64 (parity mode)
    n_devices: int = 0               # 0: min(visible GPUs, n_workers)
    global_allreduce: str = "ordered"   # ordered (reference order, push exchange) | nccl
    gemm: str = "auto"               # auto | simt | tcgen05
    data: str = "device"             # device | host
    model: str = "mlp"               # mlp | synthetic_gradient
    record_phases: bool = False
    csgd_nccl: bool = False
    synthetic_params: int = 0


@dataclass
class TrainConfig:
    """executors.hpp:218-242 (+ DataSpec :203-211, HyperParams optimizer.hpp:16-33, DelaySpec :213-216)."""

    algorithm: str = "sequential"
    n_workers: int = 1
    n_groups: int = 1
    layer_sizes: List[int] = field(default_factory=lambda: [32, 16, 10])
    n_samples: int = 5000
    n_features: int = 32
    n_classes: int = 10
    spread: float = 10.0
    mode: str = "momentum"
    base_lr: float = 0.1
    momentum: float = 0.9
    weight_decay: float = 1e-4
    warmup_epochs: float = 5.0
    decay_every_epochs: int = 30
    decay_factor: float = 0.1
    local_batch: int = 64
    epochs: int = 1
    iterations: int = 0
    seed: int = 42
    init_scale: float = 0.05
    io_delay_s: float = 0.0
    global_link_delay_s: float = 0.0
    collective_timeout_s: float = 30.0
    record_history: bool = False
    shared_minibatch: bool = True
    b200: B200Options = field(default_factory=B200Options)

    @property
    def global_batch(self) -> int:
        return self.local_batch * self.n_workers

    @property
    def n_params(self) -> int:
        if self.b200.model == "synthetic_gradient":
            return self.b200.synthetic_params
        L = self.layer_sizes
        return sum(L[k] * L[k + 1] + L[k + 1] for k in range(len(L) - 1))

    def resolve_iterations(self, dataset_size: Optional[int] = None) -> int:
        n = self.n_samples if dataset_size is None else dataset_size
        if self.iterations > 0:
            return self.iterations
        return self.epochs * (n // self.global_batch)

    def epoch_float(self, t: int, dataset_size: Optional[int] = None) -> float:
        n = self.n_samples if dataset_size is None else dataset_size
        return float(t) * float(self.global_batch) / float(n)

    def to_c(self):
        """Return (Config, keepalive) — keepalive owns the layer array the struct points to."""
        cfg = N.Config()
        N.check(N.lib.lsgd_b200_config_init(C.byref(cfg)))
        ls = (C.c_int32 * len(self.layer_sizes))(*self.layer_sizes)
        b = self.b200
        vals = dict(
            algorithm=_enum(ALGORITHMS, self.algorithm, "algorithm"), n_workers=self.n_workers,
            n_groups=self.n_groups, n_layers=len(self.layer_sizes), layer_sizes=C.cast(ls, C.POINTER(C.c_int32)),
            n_samples=self.n_samples, n_features=self.n_features, n_classes=self.n_classes, spread=self.spread,
            mode=_enum({"plain": N.PLAIN, "momentum": N.MOMENTUM}, self.mode, "optim.mode"), base_lr=self.base_lr,
            momentum=self.momentum, weight_decay=self.weight_decay, warmup_epochs=self.warmup_epochs,
            decay_every_epochs=self.decay_every_epochs, decay_factor=self.decay_factor,
            local_batch=self.local_batch, epochs=self.epochs, iterations=self.iterations, seed=self.seed,
            init_scale=self.init_scale, io_delay_s=self.io_delay_s, global_link_delay_s=self.global_link_delay_s,
            collective_timeout_s=self.collective_timeout_s, record_history=int(self.record_history),
            shared_minibatch=int(self.shared_minibatch),
            dtype=_enum({"fp32": N.FP32, "fp64": N.FP64}, b.dtype, "b200.dtype"), n_devices=b.n_devices,
            global_algo=_enum({"nccl": N.GLOBAL_NCCL, "ordered": N.GLOBAL_ORDERED}, b.global_allreduce,
                              "b200.global_allreduce"),
            gemm=_enum({"auto": N.GEMM_AUTO, "simt": N.GEMM_SIMT, "tcgen05": N.GEMM_TC}, b.gemm, "b200.gemm"),
            data_source=_enum({"device": N.DATA_DEVICE, "host": N.DATA_HOST}, b.data, "b200.data"),
            model=_enum({"mlp": N.MODEL_MLP, "synthetic_gradient": N.MODEL_SYNTHETIC_GRADIENT}, b.model,
                        "b200.model"),
            record_phases=int(b.record_phases), csgd_nccl=int(b.csgd_nccl), synthetic_params=b.synthetic_params,
        )
        for k, v in vals.items():
            setattr(cfg, k, v)
        return cfg, ls

    def validate(self) -> None:
        cfg, _keep = self.to_c()
        N.check(N.lib.lsgd_b200_config_validate(C.byref(cfg)))


def _enum(table, value, key):
    if value not in table:
        raise N.ConfigError(f"{key}: expected {'|'.join(table)}, got '{value}'")
    return table[value]


@dataclass
class TrainResult:
    """executors.hpp:287-296 (worker-0 view) plus per-worker finals and phase spans."""

    initial_params: np.ndarray
    final_params: np.ndarray
    loss_history: np.ndarray
    lr_history: np.ndarray
    param_history: Optional[np.ndarray]
    worker_finals: np.ndarray
    version_at_compute: np.ndarray
    phase_spans: Optional[np.ndarray]
    total_wall_s: float
    throughput_sps: float
    gpu_launches: int


def _ptr(a, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


def init_params(layer_sizes, seed, scale) -> np.ndarray:
    L = (C.c_int32 * len(layer_sizes))(*layer_sizes)
    P = N.lib.lsgd_b200_n_params(len(layer_sizes), L)
    w = np.zeros(P)
    N.check(N.lib.lsgd_b200_init_params(len(layer_sizes), L, seed, scale, w.ctypes.data))
    return w


def run_train(cfg: TrainConfig) -> TrainResult:
    """run_train (executors.hpp:138) on the b200 backend."""
    c, _keep = cfg.to_c()
    T = cfg.resolve_iterations()
    P = cfg.n_params
    Nw = cfg.n_workers
    want_hist = cfg.record_history
    out = dict(
        final_params=np.zeros(P), loss=np.zeros(T), lr=np.zeros(T),
        history=np.zeros((T + 1, P)) if want_hist else None, worker_finals=np.zeros((Nw, P)),
        version=np.zeros((Nw, T), dtype=np.int64),
        phases=np.zeros((Nw, T, 6, 2)) if cfg.b200.record_phases else None,
    )
    res = N.Result(_ptr(out["final_params"]), _ptr(out["loss"]), _ptr(out["lr"]), _ptr(out["history"]),
                   _ptr(out["worker_finals"]), _ptr(out["version"], C.c_int64), _ptr(out["phases"]), 0.0, 0.0, 0)
    N.check(N.lib.lsgd_b200_run_train(C.byref(c), C.byref(res)))
    w0 = init_params(cfg.layer_sizes, cfg.seed + 1, cfg.init_scale) if cfg.b200.model == "mlp" else np.zeros(P)
    return TrainResult(w0, out["final_params"], out["loss"], out["lr"], out["history"], out["worker_finals"],
                       out["version"], out["phases"], res.total_wall_s, res.throughput_sps, res.gpu_launches)


@dataclass
class EquivalenceEntry:
    name: str
    max_rel_deviation: float = 0.0
    max_normwise_deviation: float = 0.0
    worst_iteration: int = -1
    bitwise_equal: bool = False


@dataclass
class EquivalenceReport:
    entries: list
    tolerance: float
    metric: str
    passed: bool


def compare_histories(ref_hist: np.ndarray, hist: np.ndarray, name: str) -> EquivalenceEntry:
    """executors.cpp:565-586's per-coordinate |a-b|/max(|a|,1e-8), plus the norm-wise ||a-b||/||a|| per t."""
    e = EquivalenceEntry(name)
    e.bitwise_equal = ref_hist.shape == hist.shape and bool(np.array_equal(ref_hist.view(np.uint64),
                                                                           hist.view(np.uint64)))
    dev = np.abs(ref_hist - hist) / np.maximum(np.abs(ref_hist), 1e-8)
    e.max_rel_deviation = float(dev.max()) if dev.size else 0.0
    e.worst_iteration = int(np.unravel_index(np.argmax(dev), dev.shape)[0]) if dev.size else -1
    nrm = np.linalg.norm(ref_hist - hist, axis=1) / np.maximum(np.linalg.norm(ref_hist, axis=1), 1e-300)
    e.max_normwise_deviation = float(nrm.max()) if nrm.size else 0.0
    return e


def verify_equivalence(configs: List[TrainConfig], tolerance: float = 1e-8, metric: str = "coordinate"):
    """executors.cpp:523-588. metric 'coordinate' (the reference's) or 'normwise' (fp32 parity contract)."""
    if len(configs) < 2:
        raise N.ConfigError("verify: need at least two configs")
    ref = configs[0]
    for c in configs:
        c.validate()
        if c.mode != "plain":
            raise N.ConfigError("verify: iterate comparison requires optim.mode = plain")
        if not c.shared_minibatch:
            raise N.ConfigError("verify: iterate comparison requires the shared-minibatch mode")
        for key in ("seed", "layer_sizes", "global_batch", "epochs", "iterations", "init_scale", "base_lr",
                    "warmup_epochs", "decay_every_epochs", "decay_factor", "n_samples", "n_features", "n_classes",
                    "spread"):
            if getattr(c, key) != getattr(ref, key):
                raise N.ConfigError(f"verify: configs disagree on {key}")
    hists = []
    for c in configs:
        rc = TrainConfig(**{**c.__dict__, "record_history": True})
        hists.append(run_train(rc).param_history)
    entries = []
    passed = True
    for i, (c, h) in enumerate(zip(configs, hists)):
        e = compare_histories(hists[0], h, f"{c.algorithm} N={c.n_workers} G={c.n_groups}")
        val = e.max_rel_deviation if metric == "coordinate" else e.max_normwise_deviation
        if i > 0 and val > tolerance:
            passed = False
        entries.append(e)
    return EquivalenceReport(entries, tolerance, metric, passed)


class Rank:
    """One worker of a one-process-per-GPU world (run_rank seam, executors.hpp:143-144)."""

    def __init__(self, cfg: TrainConfig, rank: int, device: int):
        self.cfg = cfg
        self._c, self._keep = cfg.to_c()
        h = C.c_void_p()
        N.check(N.lib.lsgd_b200_rank_create(C.byref(self._c), rank, device, C.byref(h)))
        self.h = h
        self.rank = rank

    @staticmethod
    def blob_size() -> int:
        n = C.c_int64()
        N.check(N.lib.lsgd_b200_rank_blob_size(C.byref(n)))
        return n.value

    def export(self) -> bytes:
        buf = C.create_string_buffer(self.blob_size())
        N.check(N.lib.lsgd_b200_rank_export(self.h, buf))
        return buf.raw

    def connect(self, blobs: List[bytes]) -> None:
        allb = b"".join(blobs)
        N.check(N.lib.lsgd_b200_rank_connect(self.h, C.c_char_p(allb)))

    def upload_dataset(self, x: np.ndarray, y: np.ndarray) -> None:
        """The caller's dataset (run_rank's `const Dataset&`, executors.hpp:143-144): x [n, d] float64, y [n]."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.int32)
        if x.ndim != 2 or y.shape != (x.shape[0],):
            raise N.ConfigError(f"upload_dataset: x must be [n, d] and y [n], got {x.shape} and {y.shape}")
        N.check(N.lib.lsgd_b200_rank_upload_dataset(self.h, x.ctypes.data, y.ctypes.data, x.shape[0], x.shape[1]))

    def step(self, n: int = 1, shard_indices: Optional[np.ndarray] = None) -> None:
        p = None
        if shard_indices is not None:
            shard_indices = np.ascontiguousarray(shard_indices, dtype=np.int32)
            p = shard_indices.ctypes.data
        N.check(N.lib.lsgd_b200_rank_step(self.h, n, p))

    def step_rows(self, x_ptr: int, y_ptr: int, n: int = 1) -> None:
        """x_ptr/y_ptr: host addresses of [n, B_loc, d] rows (config dtype) and [n, B_loc] int32 labels."""
        N.check(N.lib.lsgd_b200_rank_step_rows(self.h, n, C.c_void_p(x_ptr), C.c_void_p(y_ptr)))

    def drain(self) -> None:
        N.check(N.lib.lsgd_b200_rank_drain(self.h))

    def synchronize(self) -> None:
        N.check(N.lib.lsgd_b200_rank_synchronize(self.h))

    def last_loss(self) -> float:
        v = C.c_double()
        N.check(N.lib.lsgd_b200_rank_last_loss(self.h, C.byref(v)))
        return v.value

    def join(self) -> None:
        """Order the rank's stream after all work issued so far on its side streams (no host sync)."""
        N.check(N.lib.lsgd_b200_rank_join(self.h))

    def loss_async(self, host_pinned_ptr: int) -> int:
        """Enqueue the D2H copy of the latest applied round's loss into pinned host memory (no host sync);
        returns the element size in bytes (4 for fp32, 8 for fp64)."""
        n = C.c_int32()
        N.check(N.lib.lsgd_b200_rank_loss_async(self.h, C.c_void_p(host_pinned_ptr), C.byref(n)))
        return n.value

    def params(self) -> np.ndarray:
        w = np.zeros(self.cfg.n_params)
        N.check(N.lib.lsgd_b200_rank_get_params(self.h, w.ctypes.data, w.size))
        return w

    def history(self, n: int):
        loss, lr = np.zeros(n), np.zeros(n)
        N.check(N.lib.lsgd_b200_rank_history(self.h, loss.ctypes.data, lr.ctypes.data, n))
        return loss, lr

    def launches(self) -> int:
        v = C.c_int64()
        N.check(N.lib.lsgd_b200_rank_launches(self.h, C.byref(v)))
        return v.value

    def stream(self) -> int:
        v = C.c_void_p()
        N.check(N.lib.lsgd_b200_rank_stream(self.h, C.byref(v)))
        return v.value or 0

    def timing(self, on: bool) -> None:
        N.check(N.lib.lsgd_b200_rank_timing(self.h, int(on)))

    def kernel_time(self, family: str):
        ms, cnt = C.c_double(), C.c_int64()
        N.check(N.lib.lsgd_b200_rank_kernel_time(self.h, family.encode(), C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def close(self) -> None:
        if self.h:
            N.check(N.lib.lsgd_b200_rank_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
