"""Kernel and transport seams of the C-ABI (single GPU): batch_gradient (mlp.hpp:54), the ordered collectives
(transport.hpp:56-63) and sgd_update (optimizer.hpp:51-52), executed by the same CUDA kernels the step uses."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N

_DT = {"fp32": N.FP32, "fp64": N.FP64}
_GEMM = {"auto": N.GEMM_AUTO, "simt": N.GEMM_SIMT, "tcgen05": N.GEMM_TC}


def batch_gradient(layer_sizes, w, x, y, idx, dtype="fp64", gemm="auto"):
    L = (C.c_int32 * len(layer_sizes))(*layer_sizes)
    w = np.ascontiguousarray(w, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    g = np.zeros(w.size)
    loss = C.c_double()
    N.check(N.lib.lsgd_b200_batch_gradient(len(layer_sizes), L, _DT[dtype], _GEMM[gemm], w.ctypes.data, y.size,
                                           x.ctypes.data, y.ctypes.data, idx.ctypes.data, idx.size, g.ctypes.data,
                                           C.byref(loss)))
    return g, loss.value


def collective(op, contributions, root=0, dtype="fp64"):
    c = np.ascontiguousarray(contributions, dtype=np.float64)
    out = np.full_like(c, np.nan)
    code = {"reduce": 0, "broadcast": 1, "allreduce": 2}[op]
    N.check(N.lib.lsgd_b200_collective(code, _DT[dtype], c.shape[0], root, c.shape[1], c.ctypes.data,
                                       out.ctypes.data))
    return out


def sgd_update(w, delta, velocity, mode, momentum, weight_decay, lr, dtype="fp64"):
    w = np.array(w, dtype=np.float64)
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    v = None if velocity is None else np.array(velocity, dtype=np.float64)
    m = {"plain": N.PLAIN, "momentum": N.MOMENTUM}[mode]
    N.check(N.lib.lsgd_b200_sgd_update(_DT[dtype], w.size, w.ctypes.data, delta.ctypes.data,
                                       v.ctypes.data if v is not None else None, m, momentum, weight_decay, lr))
    return w, v
