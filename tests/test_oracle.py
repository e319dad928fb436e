"""The oracle is pinned before it is trusted (CPU only).

Checks oracle/lsgd_oracle.c (the C restatement) against
  * the values asserted by the reference's own test suites (tests/golden/reference_tests.json), and
  * fixtures produced by the unmodified reference library (tests/golden/ref_fixtures.*).
"""
import json
import os

import numpy as np
import pytest

from oracle import Oracle, TrainSpec, fnv1a64

GOLD = os.path.join(os.path.dirname(__file__), "golden")
REFT = json.load(open(os.path.join(GOLD, "reference_tests.json")))
META = json.load(open(os.path.join(GOLD, "ref_fixtures.json")))
FX = np.load(os.path.join(GOLD, "ref_fixtures.npz"))


@pytest.fixture(scope="module")
def port():
    return Oracle("port")


def test_splitmix_reference_vectors(port):
    got = [f"{v:016x}" for v in port.splitmix(0, 2)]
    assert got == REFT["splitmix_seed0"]["values"]
    assert np.array_equal(port.splitmix(42, 64), FX["splitmix_42"])


def test_fisher_yates_and_partition(port):
    draws, _ = port.sampler(8, 42, 4, 2)
    assert draws.tolist() == REFT["fisher_yates_seed42_n8"]["draws"]
    p = REFT["partition"]
    assert port.partition(p["input"], p["n_workers"]).tolist() == p["shards"]
    with pytest.raises(ValueError):
        port.partition(list(range(p["bad_size"])), p["n_workers"])
    cfg1, _ = port.sampler(5000, 44, 64, 100)
    assert np.array_equal(cfg1, FX["sampler_cfg1"])
    dl, ep = port.sampler(10, 3, 4, 3)
    assert np.array_equal(dl, FX["sampler_droplast"]) and ep == META["sampler_droplast_epochs"] == 2
    rp, _ = port.sampler(10, 4, 8, 5, with_replacement=True)
    assert np.array_equal(rp, FX["sampler_repl"])


def test_synthetic_dataset_bitwise(port):
    x, y = port.generate_synthetic(42, 5000, 32, 10, 10.0)
    assert fnv1a64(x) == META["data_5000x32_fnv"]
    assert np.array_equal(x[:64], FX["data_x_head"]) and np.array_equal(y[:64], FX["data_y_head"])
    xo, yo = port.generate_synthetic(7, 9, 5, 3, 2.5)
    assert np.array_equal(xo, FX["data_odd_x"]) and np.array_equal(yo, FX["data_odd_y"])


def test_layout_and_closed_form_gradient(port):
    lay = REFT["layout_4_3_2"]
    assert TrainSpec(layer_sizes=[4, 3, 2]).n_params == lay["n_params"]
    cf = REFT["closed_form_gradient"]
    g, loss = port.batch_gradient([2, 2], np.zeros(6), np.array([cf["x"]]), np.array([cf["label"]]), [0])
    assert np.allclose(g, cf["grad"], rtol=0, atol=1e-15) and abs(loss - cf["loss"]) < 1e-12


def test_batch_gradient_bitwise(port):
    w0 = port.init_params([32, 16, 10], 43, 0.05)
    assert np.array_equal(w0, FX["init_w0"])
    x, y = port.generate_synthetic(42, 5000, 32, 10, 10.0)
    g, loss = port.batch_gradient([32, 16, 10], w0, x, y, FX["sampler_cfg1"][0])
    assert np.array_equal(g, FX["grad_w0_batch0"]) and loss == FX["loss_w0_batch0"][0]
    g, loss = port.batch_gradient([8, 12, 7, 5], FX["deep_w"], FX["deep_x"], FX["deep_y"], FX["deep_idx"])
    assert np.array_equal(g, FX["deep_grad"]) and loss == FX["deep_loss"][0]


def test_update_and_lr(port):
    u = REFT["update_plain"]
    w, _ = port.sgd_update([u["w"]], [u["delta"]], None, "plain", 0.9, 1e-4, u["lr"])
    assert abs(w[0] - u["w_new"]) < 1e-15
    u = REFT["update_momentum"]
    w, v = port.sgd_update([u["w"]], [u["delta"]], [0.0], "momentum", u["momentum"], u["weight_decay"], u["lr"])
    assert abs(w[0] - u["w_new"]) < 1e-12 and abs(v[0] - u["v_new"]) < 1e-12
    for nw, lb, ep, want in REFT["lr_points"]["cases"]:
        assert abs(port.learning_rate(0.1, 5.0, 30, 0.1, nw, lb, ep) - want) <= 1e-12


def test_ordered_collectives_bitwise(port):
    r = REFT["ordered_reduce"]
    assert port.collective("reduce", r["contributions"])[0].tolist() == r["sum"]
    c = FX["coll_contrib"]
    assert np.array_equal(port.collective("reduce", c, root=2)[2], FX["coll_reduce_root2"])
    assert np.array_equal(port.collective("allreduce", c)[3], FX["coll_allreduce"])


@pytest.mark.parametrize("name", sorted(META["hashes"]))
def test_training_history_bitwise(port, name):
    spec = TrainSpec(**META["specs"][name])
    out = port.run_train(spec, history=True, workers=True)
    assert fnv1a64(out["final_params"]) == META["hashes"][name]
    assert np.array_equal(out["loss"], FX[f"{name}_loss"])
    assert np.array_equal(out["lr"], FX[f"{name}_lr"])
    assert np.array_equal(out["history"][FX[f"{name}_hist_rows"]], FX[f"{name}_hist"])
    assert (out["version_at_compute"] == np.arange(spec.resolve_iterations())[None, :]).all()


def test_survey_hashes_and_degenerate_invariants():
    h = META["hashes"]
    s = REFT["survey_hashes"]
    for k in ("seq", "lsgd_1x1", "lsgd_2x2", "lsgd_2x4", "lsgd_4x2", "lsgd_1x8"):
        assert h[k] == s[k]
    assert h["csgd_1"] == h["seq"] == h["lsgd_1x1"]          # acceptance.cpp:87-105
    assert h["lsgd_1x4"] == h["csgd_4"] and h["lsgd_1x8"] == h["csgd_8"]  # test_executors.cpp:136-145
    assert META["loss_last"]["seq"] == s["seq_loss99"]
    assert META["loss_last"]["lsgd_2x2_mom"] == s["lsgd_2x2_mom_loss99"]


def test_port_matches_reference_live():
    """When the reference build is present (always in the build container), compare live."""
    try:
        ref = Oracle("reference")
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built")
    spec = TrainSpec(algorithm="lsgd", n_workers=6, n_groups=3, local_batch=8, iterations=25, mode="momentum",
                     layer_sizes=[32, 20, 12, 10])
    a = Oracle("port").run_train(spec)
    b = ref.run_train(spec)
    assert fnv1a64(a["final_params"]) == fnv1a64(b["final_params"])
