"""ctypes binding of ``include/lsgd_b200.h`` (the C-ABI of ``liblsgd_b200.so``, built in-tree for sm_100a).

There is no CPU fallback: the first use of ``lib`` fails loudly when the shared library is missing, and every
compute entry point raises when no sm_100 device is visible. The library is loaded lazily (module ``__getattr__``)
so that ``__graft_entry__.build()`` can import the package's build helper before the library exists.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblsgd_b200.so")

OK, ERR_RUNTIME, ERR_CONFIG, ERR_TRANSPORT = 0, 1, 2, 3
SEQUENTIAL, CSGD, LSGD = 0, 1, 2
PLAIN, MOMENTUM = 0, 1
FP32, FP64 = 0, 1
GLOBAL_NCCL, GLOBAL_ORDERED = 0, 1
GEMM_AUTO, GEMM_SIMT, GEMM_TC = 0, 1, 2
DATA_DEVICE, DATA_HOST = 0, 1
MODEL_MLP, MODEL_SYNTHETIC_GRADIENT = 0, 1


class LsgdError(RuntimeError):
    """lsgd::Error (common.hpp:16)."""


class ConfigError(LsgdError):
    """lsgd::ConfigError (common.hpp:21)."""


class TransportError(LsgdError):
    """lsgd::TransportError (common.hpp:26)."""


class Config(C.Structure):
    _fields_ = [
        ("algorithm", C.c_int32), ("n_workers", C.c_int32), ("n_groups", C.c_int32), ("n_layers", C.c_int32),
        ("layer_sizes", C.POINTER(C.c_int32)), ("n_samples", C.c_int64), ("n_features", C.c_int32),
        ("n_classes", C.c_int32), ("spread", C.c_double), ("mode", C.c_int32), ("base_lr", C.c_double),
        ("momentum", C.c_double), ("weight_decay", C.c_double), ("warmup_epochs", C.c_double),
        ("decay_every_epochs", C.c_int32), ("decay_factor", C.c_double), ("local_batch", C.c_int32),
        ("epochs", C.c_int32), ("iterations", C.c_int64), ("seed", C.c_uint64), ("init_scale", C.c_double),
        ("io_delay_s", C.c_double), ("global_link_delay_s", C.c_double), ("collective_timeout_s", C.c_double),
        ("record_history", C.c_int32), ("shared_minibatch", C.c_int32), ("dtype", C.c_int32),
        ("n_devices", C.c_int32), ("global_algo", C.c_int32), ("gemm", C.c_int32), ("data_source", C.c_int32),
        ("model", C.c_int32), ("record_phases", C.c_int32), ("csgd_nccl", C.c_int32),
        ("synthetic_params", C.c_int64),
    ]


class Result(C.Structure):
    _fields_ = [
        ("final_params", C.POINTER(C.c_double)), ("loss", C.POINTER(C.c_double)), ("lr", C.POINTER(C.c_double)),
        ("history", C.POINTER(C.c_double)), ("worker_finals", C.POINTER(C.c_double)),
        ("version_at_compute", C.POINTER(C.c_int64)), ("phase_spans", C.POINTER(C.c_double)),
        ("total_wall_s", C.c_double), ("throughput_sps", C.c_double), ("gpu_launches", C.c_int64),
    ]


_P = C.c_void_p
_SIGNATURES = {
    "lsgd_b200_last_error": ([], C.c_char_p),
    "lsgd_b200_version": ([], C.c_char_p),
    "lsgd_b200_config_init": ([C.POINTER(Config)], C.c_int),
    "lsgd_b200_config_validate": ([C.POINTER(Config)], C.c_int),
    "lsgd_b200_device_count": ([_P], C.c_int),
    "lsgd_b200_splitmix": ([C.c_uint64, C.c_int64, _P], C.c_int),
    "lsgd_b200_generate_synthetic": ([C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_double, _P, _P], C.c_int),
    "lsgd_b200_init_params": ([C.c_int32, _P, C.c_uint64, C.c_double, _P], C.c_int),
    "lsgd_b200_n_params": ([C.c_int32, _P], C.c_int64),
    "lsgd_b200_minibatch_indices": ([C.POINTER(Config), C.c_int64, C.c_int64, _P], C.c_int),
    "lsgd_b200_learning_rate": ([C.POINTER(Config), C.c_int64, _P], C.c_int),
    "lsgd_b200_topology": ([C.POINTER(Config), _P, _P, _P], C.c_int),
    "lsgd_b200_run_train": ([C.POINTER(Config), C.POINTER(Result)], C.c_int),
    "lsgd_b200_rank_create": ([C.POINTER(Config), C.c_int32, C.c_int32, _P], C.c_int),
    "lsgd_b200_rank_blob_size": ([_P], C.c_int),
    "lsgd_b200_rank_export": ([_P, _P], C.c_int),
    "lsgd_b200_rank_connect": ([_P, _P], C.c_int),
    "lsgd_b200_rank_upload_dataset": ([_P, _P, _P, C.c_int64, C.c_int32], C.c_int),
    "lsgd_b200_rank_step": ([_P, C.c_int64, _P], C.c_int),
    "lsgd_b200_rank_step_rows": ([_P, C.c_int64, _P, _P], C.c_int),
    "lsgd_b200_rank_drain": ([_P], C.c_int),
    "lsgd_b200_rank_synchronize": ([_P], C.c_int),
    "lsgd_b200_rank_last_loss": ([_P, _P], C.c_int),
    "lsgd_b200_rank_loss_async": ([_P, _P, _P], C.c_int),
    "lsgd_b200_rank_join": ([_P], C.c_int),
    "lsgd_b200_rank_get_params": ([_P, _P, C.c_int64], C.c_int),
    "lsgd_b200_rank_set_params": ([_P, _P, C.c_int64], C.c_int),
    "lsgd_b200_rank_history": ([_P, _P, _P, C.c_int64], C.c_int),
    "lsgd_b200_rank_launches": ([_P, _P], C.c_int),
    "lsgd_b200_rank_stream": ([_P, _P], C.c_int),
    "lsgd_b200_rank_kernel_time": ([_P, C.c_char_p, _P, _P], C.c_int),
    "lsgd_b200_rank_timing": ([_P, C.c_int32], C.c_int),
    "lsgd_b200_rank_destroy": ([_P], C.c_int),
    "lsgd_b200_batch_gradient": ([C.c_int32, _P, C.c_int32, C.c_int32, _P, C.c_int64, _P, _P, _P, C.c_int64, _P, _P],
                                 C.c_int),
    "lsgd_b200_collective": ([C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, _P, _P], C.c_int),
    "lsgd_b200_sgd_update": ([C.c_int32, C.c_int64, _P, _P, _P, C.c_int32, C.c_double, C.c_double, C.c_double],
                             C.c_int),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_LIB = None


def get_lib():
    """The loaded liblsgd_b200.so (loaded on first use; ImportError when it has not been built)."""
    global _LIB
    if _LIB is None:
        _LIB = _load()
    return _LIB


def __getattr__(name):
    if name == "lib":
        return get_lib()
    raise AttributeError(name)


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = get_lib().lsgd_b200_last_error().decode(errors="replace")
    raise {ERR_CONFIG: ConfigError, ERR_TRANSPORT: TransportError}.get(rc, LsgdError)(msg)


def exported_symbols():
    """Every symbol include/lsgd_b200.h declares (for the loads-and-exports test)."""
    return sorted(_SIGNATURES)
