"""CPU checks of the bench contract helpers (no GPU): the workloads are BASELINE's configs with the documented
layouts, and the reference arm's bounded cfg3 sample keeps the same layout as the b200 arm."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("n,groups,layout", [(1, None, (1, 1)), (2, None, (2, 1)), (4, None, (2, 2)),
                                             (8, None, (2, 4)), (4, 1, (1, 4)), (4, 4, (4, 1))])
def test_cfg3_workload_layouts(n, groups, layout):
    cfg = bench.workload("cfg3", n, None, "lsgd", groups=groups)
    assert cfg.layer_sizes == [4096, 8192, 8192, 512] and cfg.local_batch == 512
    assert (cfg.n_groups, cfg.n_workers // cfg.n_groups) == layout
    assert cfg.n_params == 4096 * 8192 + 8192 + 8192 * 8192 + 8192 + 8192 * 512 + 512
    assert cfg.b200.global_allreduce == "ordered"


def test_csgd_is_flat_and_bad_layouts_are_rejected():
    cfg = bench.workload("cfg3", 4, None, "csgd")
    assert cfg.n_groups == 1 and cfg.b200.csgd_nccl
    with pytest.raises(SystemExit):
        bench.workload("cfg3", 4, None, "lsgd", groups=3)


def test_synthetic_gradient_workload():
    cfg = bench.workload("cfg4", 4, None, "lsgd")
    assert cfg.b200.model == "synthetic_gradient" and cfg.b200.synthetic_params == 25_600_000
