"""TEST INFRASTRUCTURE — ctypes bindings for the CPU oracle and the reference build.

Two interchangeable backends with one Python API:

* ``Oracle("port")``      -> ``oracle/liblsgd_oracle.so``, the plain-C restatement (lsgd_oracle.c);
* ``Oracle("reference")`` -> ``oracle/_ref/liblsgd_ref.so``, the UNMODIFIED reference sources
  (/root/reference/proj/src) compiled by ``oracle/Makefile`` with ``ref_harness.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import this
package, and only as the checker. The product (``paper_1906_05936_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liblsgd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblsgd_ref.so")

ALGORITHMS = {"sequential": 0, "csgd": 1, "lsgd": 2}


class _Config(C.Structure):
    # identical layout in ref_harness.cpp (lsgd_ref_config) and lsgd_oracle.c (lo_config)
    _fields_ = [
        ("algorithm", C.c_int), ("n_workers", C.c_int), ("n_groups", C.c_int), ("n_layers", C.c_int),
        ("layer_sizes", C.POINTER(C.c_int)), ("n_samples", C.c_int64), ("n_features", C.c_int),
        ("n_classes", C.c_int), ("spread", C.c_double), ("mode", C.c_int), ("base_lr", C.c_double),
        ("momentum", C.c_double), ("weight_decay", C.c_double), ("warmup_epochs", C.c_double),
        ("decay_every_epochs", C.c_int), ("decay_factor", C.c_double), ("local_batch", C.c_int),
        ("epochs", C.c_int), ("iterations", C.c_int64), ("seed", C.c_uint64), ("init_scale", C.c_double),
        ("io_delay_s", C.c_double), ("global_link_delay_s", C.c_double), ("shared_minibatch", C.c_int),
    ]


class _Result(C.Structure):
    _fields_ = [
        ("final_params", C.POINTER(C.c_double)), ("loss", C.POINTER(C.c_double)),
        ("lr", C.POINTER(C.c_double)), ("history", C.POINTER(C.c_double)),
        ("worker_finals", C.POINTER(C.c_double)), ("version_at_compute", C.POINTER(C.c_int64)),
        ("phase_spans", C.POINTER(C.c_double)), ("total_wall_s", C.c_double),
        ("throughput_sps", C.c_double),
    ]


@dataclass
class TrainSpec:
    """Python mirror of the reference TrainConfig (proj/include/lsgd/executors.hpp:218-242)."""

    algorithm: str = "lsgd"
    n_workers: int = 1
    n_groups: int = 1
    layer_sizes: list = field(default_factory=lambda: [32, 16, 10])
    n_samples: int = 5000
    n_features: int = 32
    n_classes: int = 10
    spread: float = 10.0
    mode: str = "plain"
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
    shared_minibatch: bool = True

    @property
    def n_params(self) -> int:
        L = self.layer_sizes
        return sum(L[k] * L[k + 1] + L[k + 1] for k in range(len(L) - 1))

    def resolve_iterations(self) -> int:
        if self.iterations > 0:
            return self.iterations
        return self.epochs * (self.n_samples // (self.local_batch * self.n_workers))

    def to_c(self):
        ls = (C.c_int * len(self.layer_sizes))(*self.layer_sizes)
        c = _Config(
            ALGORITHMS[self.algorithm], self.n_workers, self.n_groups, len(self.layer_sizes), ls,
            self.n_samples, self.n_features, self.n_classes, self.spread,
            0 if self.mode == "plain" else 1, self.base_lr, self.momentum, self.weight_decay,
            self.warmup_epochs, self.decay_every_epochs, self.decay_factor, self.local_batch,
            self.epochs, self.iterations, self.seed, self.init_scale, self.io_delay_s,
            self.global_link_delay_s, 1 if self.shared_minibatch else 0,
        )
        return c, ls


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def build() -> None:
    """Compile the oracle restatement (and the reference library when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class Oracle:
    def __init__(self, kind: str = "port"):
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} is missing (reference build unavailable)")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.pfx = "lo_" if kind == "port" else "lsgd_ref_"

    def _f(self, name):
        return getattr(self.lib, self.pfx + name)

    # ---- primitives -------------------------------------------------------------------------
    def splitmix(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.uint64)
        f = self._f("splitmix")
        f.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        f(seed, n, out.ctypes.data)
        return out

    def generate_synthetic(self, seed, n, d, c, spread):
        x = np.zeros((n, d), dtype=np.float64)
        y = np.zeros(n, dtype=np.int32)
        f = self._f("generate_synthetic")
        f.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_void_p]
        rc = f(seed, n, d, c, spread, x.ctypes.data, y.ctypes.data)
        if rc:
            raise ValueError("generate_synthetic rejected its arguments")
        return x, y

    def sampler(self, n, seed, size, n_draws, with_replacement=False):
        out = np.zeros(size * n_draws, dtype=np.int32)
        ep = C.c_int64(0)
        f = self._f("sampler")
        f.argtypes = [C.c_int64, C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
        rc = f(n, seed, size, n_draws, int(with_replacement), out.ctypes.data, C.byref(ep))
        if rc:
            raise ValueError("sampler draw rejected")
        return out.reshape(n_draws, size), ep.value

    def partition(self, idx, n_workers):
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        out = np.zeros_like(idx)
        f = self._f("partition")
        f.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        if f(idx.ctypes.data, idx.size, n_workers, out.ctypes.data):
            raise ValueError("partition: size not divisible by n_workers")
        return out.reshape(n_workers, -1)

    def init_params(self, layers, seed, scale):
        L = (C.c_int * len(layers))(*layers)
        P = sum(layers[k] * layers[k + 1] + layers[k + 1] for k in range(len(layers) - 1))
        w = np.zeros(P, dtype=np.float64)
        f = self._f("init_params")
        f.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_double, C.c_void_p]
        if f(len(layers), L, seed, scale, w.ctypes.data):
            raise ValueError("init_params rejected")
        return w

    def batch_gradient(self, layers, w, x, y, idx):
        L = (C.c_int * len(layers))(*layers)
        w = np.ascontiguousarray(w, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.int32)
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        g = np.zeros(w.size, dtype=np.float64)
        loss = C.c_double(0)
        f = self._f("batch_gradient")
        if self.kind == "port":
            f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                          C.c_int64, C.c_void_p, C.c_void_p]
            rc = f(len(layers), L, w.ctypes.data, y.size, x.ctypes.data, y.ctypes.data, idx.ctypes.data,
                   idx.size, g.ctypes.data, C.byref(loss))
        else:
            f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                          C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
            rc = f(len(layers), L, w.ctypes.data, y.size, x.ctypes.data, y.ctypes.data, idx.ctypes.data,
                   idx.size, 1, g.ctypes.data, C.byref(loss))
        if rc:
            raise ValueError("batch_gradient rejected its batch")
        return g, loss.value

    def learning_rate(self, base_lr, warmup, decay_every, decay_factor, n_workers, local_batch, epoch):
        f = self._f("learning_rate")
        if self.kind == "port":
            f.restype = C.c_double
            f.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double]
            return f(base_lr, warmup, decay_every, decay_factor, n_workers, local_batch, epoch)
        out = C.c_double(0)
        f.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, C.c_void_p]
        if f(base_lr, warmup, decay_every, decay_factor, n_workers, local_batch, epoch, C.byref(out)):
            raise ValueError("learning_rate rejected")
        return out.value

    def sgd_update(self, w, delta, v, mode, momentum, weight_decay, lr):
        w = np.array(w, dtype=np.float64)
        delta = np.ascontiguousarray(delta, dtype=np.float64)
        v = None if v is None else np.array(v, dtype=np.float64)
        f = self._f("sgd_update")
        vp = v.ctypes.data if v is not None else None
        f.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double]
        m = 0 if mode == "plain" else 1
        if self.kind == "port" and m == 1 and v is None:
            v = np.zeros_like(w)
            vp = v.ctypes.data
        f(w.size, w.ctypes.data, delta.ctypes.data, vp, m, momentum, weight_decay, lr)
        return w, v

    def collective(self, op, contributions, root=0):
        """op: 'reduce' | 'broadcast' | 'allreduce'; contributions [world, n] float64."""
        c = np.ascontiguousarray(contributions, dtype=np.float64)
        out = np.full_like(c, np.nan)
        f = self._f("collective")
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_void_p, C.c_void_p]
        code = {"reduce": 0, "broadcast": 1, "allreduce": 2}[op]
        if f(code, c.shape[0], root, c.shape[1], c.ctypes.data, out.ctypes.data):
            raise ValueError("collective failed")
        return out

    # ---- training ------------------------------------------------------------------------------
    def run_train(self, spec: TrainSpec, history: bool = False, workers: bool = False):
        T = spec.resolve_iterations()
        P = spec.n_params
        N = spec.n_workers
        world = N + (spec.n_groups if spec.algorithm == "lsgd" else 0)
        out = {
            "final_params": np.zeros(P), "loss": np.zeros(T), "lr": np.zeros(T),
            "history": np.zeros((T + 1, P)) if history else None,
            "worker_finals": np.zeros((N, P)) if workers else None,
            "version_at_compute": np.zeros((N, T), dtype=np.int64) if workers else None,
            "phase_spans": np.zeros((world, T, 6, 2)) if (workers and self.kind == "reference") else None,
        }
        cfg, _keep = spec.to_c()
        res = _Result(
            _dp(out["final_params"]), _dp(out["loss"]), _dp(out["lr"]), _dp(out["history"]),
            _dp(out["worker_finals"]),
            out["version_at_compute"].ctypes.data_as(C.POINTER(C.c_int64)) if workers else None,
            _dp(out["phase_spans"]), 0.0, 0.0,
        )
        f = self._f("run_train")
        f.argtypes = [C.POINTER(_Config), C.POINTER(_Result)]
        rc = f(C.byref(cfg), C.byref(res))
        if rc:
            msg = ""
            if self.kind == "reference":
                self.lib.lsgd_ref_last_error.restype = C.c_char_p
                msg = self.lib.lsgd_ref_last_error().decode()
            raise RuntimeError(f"{self.kind} run_train failed (rc={rc}) {msg}")
        out["total_wall_s"] = res.total_wall_s
        out["throughput_sps"] = res.throughput_sps
        return out


def fnv1a64(a: np.ndarray) -> str:
    """fnv1a-64 of the raw bytes (the survey's golden hashes of w_100)."""
    h = 1469598103934665603
    for b in np.ascontiguousarray(a).tobytes():
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"
