"""B200-native Layered SGD synchronous update step (arXiv 1906.05936), drop-in for the reference's LSGD step.

The compute path is ``liblsgd_b200.so`` (CUDA sm_100a + NCCL, C-ABI ``include/lsgd_b200.h``); this package is
the host-side mirror of the reference's executor / config surface over that ABI.
"""
from ._native import ConfigError, LsgdError, TransportError  # noqa: F401
from .executors import (B200Options, Rank, TrainConfig, TrainResult, run_train,  # noqa: F401
                        verify_equivalence)
from .metrics import K_METRICS_HEADER, write_metrics_csv  # noqa: F401

__all__ = ["TrainConfig", "B200Options", "TrainResult", "run_train", "verify_equivalence", "Rank", "LsgdError",
           "ConfigError", "TransportError", "write_metrics_csv", "K_METRICS_HEADER"]
