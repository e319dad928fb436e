"""Per-iteration metrics CSV in the reference's exact schema.

Mirrors `write_metrics_csv` (proj/src/metrics.cpp:32-44) with the header `kMetricsHeader`
(proj/include/lsgd/metrics.hpp:12-15): one row per iteration, the six phase durations from the device-recorded
spans (CUDA events, `b200.record_phases = true`), `%.17g` floats. Attribution follows the reference
(executors.hpp:96-98, executors.cpp:343-353): worker 0's spans, except the global allreduce, which reports the
widest span over the ranks that run it (here: every slot owner).
"""
from __future__ import annotations

import numpy as np

from .executors import TrainConfig, TrainResult

K_METRICS_HEADER = ("run_id,algorithm,n_workers,n_groups,iteration,epoch,lr,loss,"
                    "t_io_s,t_compute_s,t_local_reduce_s,t_global_allreduce_s,t_broadcast_s,t_update_s,"
                    "iter_time_s,throughput_sps")
PHASES = ("io", "compute", "local_reduce", "global_allreduce", "broadcast", "update")


def _fmt(v: float) -> str:
    return "%.17g" % float(v)


def metrics_rows(cfg: TrainConfig, result: TrainResult):
    """Per-iteration (phase durations[6], iter_wall) from result.phase_spans [workers, T, 6, (begin, end)]."""
    spans = result.phase_spans
    if spans is None:
        raise ValueError("metrics need phase spans: run with cfg.b200.record_phases = True")
    T = spans.shape[1]
    rows = []
    for t in range(T):
        ph = spans[0, t]
        dur = np.maximum(ph[:, 1] - ph[:, 0], 0.0)
        if cfg.algorithm == "lsgd":  # the slowest global allreduce among the ranks that run it
            g = np.maximum(spans[:, t, 3, 1] - spans[:, t, 3, 0], 0.0)
            dur[3] = g.max()
        present = ph[:, 1] > ph[:, 0]
        begin = ph[0, 0]
        end = ph[present, 1].max() if present.any() else begin
        rows.append((dur, max(end - begin, 0.0)))
    return rows


def write_metrics_csv(path: str, run_id: str, cfg: TrainConfig, result: TrainResult) -> None:
    """The reference's metrics CSV for a run of `run_train` (exact header and column order)."""
    rows = metrics_rows(cfg, result)
    gb = cfg.global_batch
    with open(path, "w") as f:
        f.write(K_METRICS_HEADER + "\n")
        for t, (dur, wall) in enumerate(rows):
            loss = result.loss_history[t] if t < len(result.loss_history) else 0.0
            lr = result.lr_history[t] if t < len(result.lr_history) else 0.0
            thr = gb / wall if wall > 0 else 0.0
            f.write(",".join([run_id, cfg.algorithm, str(cfg.n_workers), str(cfg.n_groups), str(t),
                              _fmt(cfg.epoch_float(t)), _fmt(lr), _fmt(loss)] + [_fmt(d) for d in dur] +
                             [_fmt(wall), _fmt(thr)]) + "\n")
