"""Bit-exact host-side pieces exported by the C-ABI (no GPU needed): SplitMix64 (rng.hpp:14-51), synthetic blobs
(dataset.cpp:32-70), the minibatch/shard stream (sampler.cpp:15-57, executors.cpp:67-85), the learning-rate
schedule (optimizer.cpp:8-22) and the topology (executors.cpp:389-433)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .executors import TrainConfig


def splitmix(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    N.check(N.lib.lsgd_b200_splitmix(seed, n, out.ctypes.data))
    return out


def generate_synthetic(seed: int, n: int, d: int, c: int, spread: float):
    x = np.zeros((n, d))
    y = np.zeros(n, dtype=np.int32)
    N.check(N.lib.lsgd_b200_generate_synthetic(seed, n, d, c, spread, x.ctypes.data, y.ctypes.data))
    return x, y


def minibatch_indices(cfg: TrainConfig, t0: int, n_steps: int) -> np.ndarray:
    """[n_steps, global_batch]; worker i's shard is columns [i*B_loc, (i+1)*B_loc)."""
    c, _keep = cfg.to_c()
    out = np.zeros((n_steps, cfg.global_batch), dtype=np.int32)
    N.check(N.lib.lsgd_b200_minibatch_indices(C.byref(c), t0, n_steps, out.ctypes.data))
    return out


def learning_rate(cfg: TrainConfig, t: int) -> float:
    c, _keep = cfg.to_c()
    v = C.c_double()
    N.check(N.lib.lsgd_b200_learning_rate(C.byref(c), t, C.byref(v)))
    return v.value


def topology(cfg: TrainConfig):
    """(role[world], group[world], device_of_worker[N]); role 0 = worker, 1 = communicator."""
    c, _keep = cfg.to_c()
    world = cfg.n_workers + (cfg.n_groups if cfg.algorithm == "lsgd" else 0)
    role = np.zeros(world, dtype=np.int32)
    group = np.zeros(world, dtype=np.int32)
    dev = np.zeros(cfg.n_workers, dtype=np.int32)
    N.check(N.lib.lsgd_b200_topology(C.byref(c), role.ctypes.data, group.ctypes.data, dev.ctypes.data))
    return role, group, dev


def device_count() -> int:
    v = C.c_int32()
    N.check(N.lib.lsgd_b200_device_count(C.byref(v)))
    return v.value
