"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every symbol include/lsgd_b200.h declares,
and its host-side pieces are bit-exact against the oracle / reference goldens. No GPU needed."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_1906_05936_b200 as lsgd
from paper_1906_05936_b200 import _native as N
from paper_1906_05936_b200 import host
from paper_1906_05936_b200.config import parse_run_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INCLUDE = "/root/reference/proj/include/lsgd"  # present in the build container only (CPU tests)
GOLD = os.path.join(ROOT, "tests", "golden")
REFT = json.load(open(os.path.join(GOLD, "reference_tests.json")))
FX = np.load(os.path.join(GOLD, "ref_fixtures.npz"))
META = json.load(open(os.path.join(GOLD, "ref_fixtures.json")))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "lsgd_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lsgd_b200_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(N.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/lsgd_b200.h but not exported"
    assert set(syms) == set(N.exported_symbols())


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {N.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_splitmix_and_dataset_bitwise():
    assert [f"{v:016x}" for v in host.splitmix(0, 2)] == REFT["splitmix_seed0"]["values"]
    assert np.array_equal(host.splitmix(42, 64), FX["splitmix_42"])
    x, y = host.generate_synthetic(42, 5000, 32, 10, 10.0)
    from oracle import fnv1a64
    assert fnv1a64(x) == META["data_5000x32_fnv"]
    xo, yo = host.generate_synthetic(7, 9, 5, 3, 2.5)
    assert np.array_equal(xo, FX["data_odd_x"]) and np.array_equal(yo, FX["data_odd_y"])


def test_parallel_blob_generator_matches_sequential_reference():
    """The product generates large datasets row-parallel (SplitMix64 is a counter); bitwise vs the oracle."""
    from oracle import Oracle
    x, y = host.generate_synthetic(9, 4099, 1025, 7, 3.0)  # > 4M values: takes the threaded path, odd d
    xo, yo = Oracle("port").generate_synthetic(9, 4099, 1025, 7, 3.0)
    assert np.array_equal(x, xo) and np.array_equal(y, yo)


def test_minibatch_stream_and_shards_bitwise():
    cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=4, n_groups=2, local_batch=16, iterations=100, mode="plain")
    idx = host.minibatch_indices(cfg, 0, 100)
    assert np.array_equal(idx, FX["sampler_cfg1"])
    tail = host.minibatch_indices(cfg, 77, 5)
    assert np.array_equal(tail, FX["sampler_cfg1"][77:82])
    small = lsgd.TrainConfig(n_samples=8, n_features=32, local_batch=4, seed=40)  # sampler seed = seed + 2 = 42
    assert host.minibatch_indices(small, 0, 2).tolist() == REFT["fisher_yates_seed42_n8"]["draws"]


def test_learning_rate_reference_points():
    for nw, lb, ep, want in REFT["lr_points"]["cases"]:
        # choose n_samples so epoch_float(t=1) == ep exactly: epoch = t * gb / n
        cfg = lsgd.TrainConfig(n_workers=nw, local_batch=lb, algorithm="csgd")
        if ep == 0.0:
            assert abs(host.learning_rate(cfg, 0) - want) <= 1e-12
            continue
        gb = nw * lb
        cfg.n_samples = gb * 1000  # epoch_float(t) = t / 1000 (exact for these points)
        got = host.learning_rate(cfg, int(round(ep * 1000)))
        assert abs(got - want) <= 1e-12, (nw, lb, ep, got, want)
    cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=4, n_groups=2, local_batch=16, iterations=100)
    lrs = [host.learning_rate(cfg, t) for t in range(100)]
    assert np.array_equal(np.array(lrs), FX["lsgd_2x2_lr"])


def test_topology_matches_reference():
    t = REFT["topology_8x2"]
    cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=8, n_groups=2, n_samples=5000)
    role, group, dev = host.topology(cfg)
    assert len(role) == t["world_lsgd"]
    assert role[3] == 0 and role[8] == 1 and group[5] == t["group_5"] and group[9] == t["group_9"]
    members_1 = [r for r in range(8) if group[r] == 1] + [8 + 1]
    assert members_1 == t["local_group_1"]
    with pytest.raises(lsgd.ConfigError):
        lsgd.TrainConfig(algorithm="lsgd", n_workers=6, n_groups=4).validate()


def test_config_validation_mirrors_reference():
    lsgd.TrainConfig(algorithm="lsgd", n_workers=4, n_groups=2, local_batch=16).validate()
    bad = [
        dict(algorithm="sequential", n_workers=2),
        dict(algorithm="lsgd", n_workers=6, n_groups=4),
        dict(momentum=1.0), dict(base_lr=0.0), dict(decay_factor=1.5),
        dict(n_features=31), dict(local_batch=0), dict(n_samples=10, local_batch=64),
    ]
    for kw in bad:
        with pytest.raises(lsgd.ConfigError):
            lsgd.TrainConfig(**kw).validate()


TRAIN_LSGD_JSON = """{
  "algorithm": "lsgd", "n_workers": 4, "n_groups": 2, "local_batch": 16, "epochs": 5, "seed": 42,
  "model": {"layer_sizes": [32, 16, 10]},
  "data": {"source": "synthetic", "n_samples": 5000, "n_features": 32, "n_classes": 10, "spread": 10.0},
  "optim": {"mode": "momentum", "base_lr": 0.1, "momentum": 0.9, "weight_decay": 0.0001,
            "warmup_epochs": 5, "decay_every_epochs": 30, "decay_factor": 0.1}
}"""  # proj/configs/train_lsgd.json (BASELINE cfg1)


def test_config_parser_accepts_reference_schema_and_b200_backend():
    rc = parse_run_config(TRAIN_LSGD_JSON)
    t = rc.train
    assert (t.algorithm, t.n_workers, t.n_groups, t.local_batch, t.epochs) == ("lsgd", 4, 2, 16, 5)
    assert t.layer_sizes == [32, 16, 10] and t.mode == "momentum" and t.resolve_iterations() == 5 * (5000 // 64)
    doc = json.loads(TRAIN_LSGD_JSON)
    doc["transport"] = {"backend": "b200", "timeout_s": 5.0}
    doc["b200"] = {"dtype": "fp64", "global_allreduce": "ordered"}
    rc = parse_run_config(json.dumps(doc))
    assert rc.transport_backend == "b200" and rc.train.b200.dtype == "fp64"
    assert rc.train.collective_timeout_s == 5.0


@pytest.mark.parametrize("mutation,fragment", [
    (lambda d: d.update(bogus=1), "unknown key bogus"),
    (lambda d: d["model"].update(depth=3), "unknown key model.depth"),
    (lambda d: d["optim"].update(mode="adam"), "optim.mode"),
    (lambda d: d.update(n_workers="4"), "n_workers must be an integer"),
    (lambda d: d.pop("algorithm"), "missing required key algorithm"),
    (lambda d: d.update(transport={"backend": "mpi"}), "transport.backend"),
])
def test_config_parser_is_strict(mutation, fragment):
    doc = json.loads(TRAIN_LSGD_JSON)
    mutation(doc)
    with pytest.raises(lsgd.ConfigError, match=re.escape(fragment)):
        parse_run_config(json.dumps(doc))


def test_compute_entry_points_fail_loudly_without_gpu():
    if host.device_count() > 0:
        pytest.skip("GPU present")
    cfg = lsgd.TrainConfig(algorithm="sequential", iterations=1)
    with pytest.raises(lsgd.LsgdError):
        lsgd.run_train(cfg)


def test_metrics_csv_schema_matches_the_reference(tmp_path):
    """metrics.cpp:32-44 / metrics.hpp:12-15: exact header, one row per iteration, %.17g, the global allreduce
    attributed to the widest owner span (executors.cpp:343-353)."""
    import numpy as np
    from paper_1906_05936_b200.executors import TrainResult
    ref_header = open(os.path.join(REF_INCLUDE, "metrics.hpp")).read() if os.path.isdir(REF_INCLUDE) else None
    cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=2, n_groups=2, layer_sizes=[4, 3], n_samples=100,
                           local_batch=5, iterations=2)
    spans = np.zeros((2, 2, 6, 2))
    for t in range(2):
        for p in range(6):
            spans[:, t, p] = [t + 0.1 * p, t + 0.1 * p + 0.05]
    spans[1, 1, 3] = [1.3, 1.5]  # worker 1's global allreduce of round 1 is the widest
    res = TrainResult(np.zeros(15), np.zeros(15), np.array([2.0, 1.5]), np.array([0.1, 0.1]), None, np.zeros((2, 15)),
                      np.zeros((2, 2), dtype=np.int64), spans, 1.0, 20.0, 0)
    path = tmp_path / "m.csv"
    lsgd.write_metrics_csv(str(path), "r1", cfg, res)
    lines = path.read_text().splitlines()
    assert lines[0] == lsgd.K_METRICS_HEADER
    if ref_header is not None:
        flat = "".join(x.strip().strip('"') for x in ref_header.split("kMetricsHeader =")[1].split(";")[0].split("\n"))
        assert flat == lsgd.K_METRICS_HEADER
    assert len(lines) == 3
    row = lines[2].split(",")
    assert row[:5] == ["r1", "lsgd", "2", "2", "1"]
    assert float(row[5]) == 1 * 10 / 100  # epoch = t * global_batch / n
    assert abs(float(row[11]) - 0.2) < 1e-12  # widest global allreduce span
    assert abs(float(row[8]) - 0.05) < 1e-12 and abs(float(row[14]) - 0.55) < 1e-12


def test_library_exports_every_testing_symbol():
    text = open(os.path.join(ROOT, "include", "lsgd_b200_testing.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    syms = sorted(set(re.findall(r"\b(lsgd_b200_test_[a-z0-9_]+)\s*\(", text)))
    assert "lsgd_b200_test_exchange_kernel" in syms
    lib = ctypes.CDLL(N.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/lsgd_b200_testing.h but not exported"


def test_library_loads_without_a_driver():
    """No link-time dependency on libcuda: driver entry points (tensor maps, NVLS multicast) are resolved at run
    time, so the library loads in a driver-less build container and fails only when a GPU path runs."""
    out = os.popen(f"readelf -d {N.LIB_PATH} 2>/dev/null").read()
    assert "libcuda.so" not in out, out
