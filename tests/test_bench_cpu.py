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


def test_gpus_n_self_launches_one_process_per_rank():
    """`bench.py --gpus 2` without torchrun spawns 2 ranks that rendezvous (gloo, 127.0.0.1) and reach Rank(...);
    without a GPU each rank fails loudly and the job exits non-zero (no CPU fallback)."""
    import subprocess

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                        "--skip-cpu", "--skip-e2e"], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode != 0
    for r in range(2):
        assert f"[bench rank {r}/2] creating Rank" in p.stderr, p.stderr[-3000:]
    assert p.stdout.strip() == ""  # no bench line without a GPU
