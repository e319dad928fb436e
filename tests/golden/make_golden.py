"""Regenerate tests/golden/ from the UNMODIFIED reference library.

Run in the build container (needs /root/reference, builds oracle/_ref/liblsgd_ref.so):

    python tests/golden/make_golden.py

Writes
  * reference_tests.json -- values the reference's own doctest/acceptance suites assert (transcribed,
    with file:line), so the pins hold even where those suites cannot be built (doctest is absent);
  * ref_fixtures.npz     -- outputs of oracle/_ref (the reference's own code) on seeded inputs:
    SplitMix64 streams, synthetic data, sampler draws, batch gradients, collectives, and LSGD/CSGD/
    sequential training histories for cfg1/cfg2 shapes (plain and momentum);
  * ref_fixtures.json    -- fnv1a64 hashes of w_T for every layout, loss/lr endpoints.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Oracle, TrainSpec, build, fnv1a64  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
HIST_ROWS = [0, 1, 2, 3, 5, 10, 20, 30, 40, 50, 60, 70, 80, 90, 99, 100]


def cfg(alg, n, g, mode="plain", T=100, layers=(32, 16, 10), n_samples=5000, spread=10.0, gb=64):
    return TrainSpec(algorithm=alg, n_workers=n, n_groups=g, layer_sizes=list(layers), n_samples=n_samples,
                     n_features=layers[0], n_classes=layers[-1], spread=spread, mode=mode,
                     local_batch=gb // n, iterations=T)


# Layouts pinned by SURVEY.md §8(c) (acceptance.cpp:53-69 workload) and test_executors.cpp:15-31.
RUNS = {
    "seq": cfg("sequential", 1, 1),
    "lsgd_1x1": cfg("lsgd", 1, 1),
    "lsgd_2x2": cfg("lsgd", 4, 2),
    "lsgd_2x4": cfg("lsgd", 8, 2),
    "lsgd_4x2": cfg("lsgd", 8, 4),
    "lsgd_1x8": cfg("lsgd", 8, 1),
    "lsgd_1x4": cfg("lsgd", 4, 1),
    "csgd_4": cfg("csgd", 4, 1),
    "csgd_8": cfg("csgd", 8, 1),
    "csgd_1": cfg("csgd", 1, 1),
    "lsgd_2x2_mom": cfg("lsgd", 4, 2, "momentum"),
    "lsgd_1x1_mom": cfg("lsgd", 1, 1, "momentum"),
    "lsgd_2x4_mom": cfg("lsgd", 8, 2, "momentum"),
    "lsgd_2x1": cfg("lsgd", 2, 2),
    # test_executors.cpp base_config: 16-8-4, 512 samples, spread 6, global 32
    "exec_lsgd_4x2": cfg("lsgd", 4, 2, T=50, layers=(16, 8, 4), n_samples=512, spread=6.0, gb=32),
    "exec_csgd_4": cfg("csgd", 4, 1, T=30, layers=(16, 8, 4), n_samples=512, spread=6.0, gb=32),
}


def reference_tests():
    """Assertions of the reference suites, transcribed (file:line under /root/reference/proj)."""
    return {
        "splitmix_seed0": {"src": "tests/test_rng.cpp:10-14",
                           "values": ["e220a8397b1dcdaf", "6e789e6aa1b965f4"]},
        "fisher_yates_seed42_n8": {"src": "tests/test_dataset.cpp:146-157",
                                   "draws": [[3, 1, 6, 2], [4, 0, 7, 5]]},
        "partition": {"src": "tests/test_dataset.cpp:204-222", "input": list(range(8)), "n_workers": 4,
                      "shards": [[0, 1], [2, 3], [4, 5], [6, 7]], "bad_size": 6},
        "topology_8x2": {"src": "tests/test_executors.cpp:35-58", "world_lsgd": 10, "world_csgd": 8,
                         "local_group_1": [4, 5, 6, 7, 9], "local_root_1": 9, "comms": [8, 9],
                         "comm_root": 8, "role_3": "worker", "role_8": "communicator", "group_5": 1,
                         "group_9": 1},
        "layout_4_3_2": {"src": "tests/test_mlp.cpp:51-58", "n_params": 23, "w_off": [0, 15],
                         "b_off": [12, 21]},
        "closed_form_gradient": {"src": "tests/test_mlp.cpp:118-132", "x": [1.0, 2.0], "label": 0,
                                 "grad": [-0.5, -1.0, 0.5, 1.0, -0.5, 0.5], "loss": float(np.log(2.0))},
        "update_plain": {"src": "tests/test_optimizer.cpp:64-75", "w": 1.0, "delta": 0.5, "lr": 0.1,
                         "w_new": 0.95},
        "update_momentum": {"src": "tests/test_optimizer.cpp:77-86", "w": 1.0, "delta": 0.5, "lr": 0.1,
                            "momentum": 0.9, "weight_decay": 1e-4, "w_new": 0.94999, "v_new": 0.5001},
        "lr_points": {"src": "tests/test_optimizer.cpp:28-52; tests/acceptance.cpp:236-247",
                      "cases": [[4, 64, 10.0, 0.1], [256, 64, 10.0, 6.4], [256, 64, 2.5, 3.25],
                                [4, 64, 30.0, 0.01], [4, 64, 60.0, 0.001], [256, 64, 0.0, 0.1],
                                [4, 64, 29.999, 0.1]]},
        "ordered_reduce": {"src": "tests/test_transport.cpp:135-146",
                           "contributions": [[1, 2], [3, 4], [5, 6]], "sum": [9, 12]},
        "survey_hashes": {"src": "SURVEY.md §8(c) (in-container run of the reference)",
                          "seq": "97453412abaaa354", "lsgd_1x1": "97453412abaaa354",
                          "lsgd_2x2": "c7bb76ccc1d0a18c", "lsgd_2x4": "80299b09e572b181",
                          "lsgd_4x2": "6edac59405aee358", "lsgd_1x8": "56aafae02322f360",
                          "seq_loss0": 2.3003440371632604, "seq_loss99": 0.026929955450059953,
                          "lsgd_2x2_mom_loss99": 8.0337581514489109e-06},
    }


def main():
    build()
    ref = Oracle("reference")
    fx = {}
    meta = {"hashes": {}, "loss_last": {}, "specs": {}}

    fx["splitmix_42"] = ref.splitmix(42, 64)
    fx["splitmix_0"] = ref.splitmix(0, 8)
    x, y = ref.generate_synthetic(42, 5000, 32, 10, 10.0)
    fx["data_x_head"] = x[:64]
    fx["data_y_head"] = y[:64]
    meta["data_5000x32_fnv"] = fnv1a64(x)
    xo, yo = ref.generate_synthetic(7, 9, 5, 3, 2.5)  # odd feature count: discarded Box-Muller sibling
    fx["data_odd_x"], fx["data_odd_y"] = xo, yo
    fx["sampler_cfg1"], _ = ref.sampler(5000, 44, 64, 100)
    fx["sampler_droplast"], ep = ref.sampler(10, 3, 4, 3)
    meta["sampler_droplast_epochs"] = ep
    fx["sampler_repl"], _ = ref.sampler(10, 4, 8, 5, with_replacement=True)

    layers = [32, 16, 10]
    w0 = ref.init_params(layers, 43, 0.05)
    fx["init_w0"] = w0
    g, loss = ref.batch_gradient(layers, w0, x, y, fx["sampler_cfg1"][0])
    fx["grad_w0_batch0"], fx["loss_w0_batch0"] = g, np.array([loss])
    deep = [8, 12, 7, 5]
    wd = ref.init_params(deep, 5, 0.4)
    xd, yd = ref.generate_synthetic(11, 40, 8, 5, 3.0)
    idx = np.array([3, 17, 0, 39, 22, 5, 5, 11], dtype=np.int32)
    gd, ld = ref.batch_gradient(deep, wd, xd, yd, idx)
    fx["deep_w"], fx["deep_x"], fx["deep_y"], fx["deep_idx"] = wd, xd, yd, idx
    fx["deep_grad"], fx["deep_loss"] = gd, np.array([ld])

    rng = np.random.default_rng(3)
    contrib = rng.standard_normal((5, 64)) * np.array([1e-8, 1.0, 1e8, -3.0, 0.5])[:, None]
    fx["coll_contrib"] = contrib
    fx["coll_reduce_root2"] = ref.collective("reduce", contrib, root=2)[2]
    fx["coll_allreduce"] = ref.collective("allreduce", contrib)[0]

    for name, spec in RUNS.items():
        out = ref.run_train(spec, history=True, workers=True)
        meta["hashes"][name] = fnv1a64(out["final_params"])
        meta["loss_last"][name] = float(out["loss"][-1])
        meta["specs"][name] = spec.__dict__
        fx[f"{name}_loss"] = out["loss"]
        fx[f"{name}_lr"] = out["lr"]
        rows = [r for r in HIST_ROWS if r < out["history"].shape[0]]
        fx[f"{name}_hist"] = out["history"][rows]
        fx[f"{name}_hist_rows"] = np.array(rows)
        for wk in range(spec.n_workers):
            assert fnv1a64(out["worker_finals"][wk]) == meta["hashes"][name], "replicas diverged"
    np.savez_compressed(os.path.join(OUT, "ref_fixtures.npz"), **fx)
    with open(os.path.join(OUT, "ref_fixtures.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    with open(os.path.join(OUT, "reference_tests.json"), "w") as f:
        json.dump(reference_tests(), f, indent=1)
    print("wrote", sorted(fx)[:5], "...", len(fx), "arrays;", meta["hashes"])


if __name__ == "__main__":
    main()
