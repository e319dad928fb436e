"""Wall time per block of LSGD vs CSGD with injected io / link delays (test_executors.cpp:195-220 setting)."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1906_05936_b200 as lsgd  # noqa: E402

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 4
for (alg, G), rec, (io, link) in itertools.product([("csgd", 1), ("lsgd", 2)], [False, True],
                                                   [(0.0, 0.0), (0.020, 0.0), (0.0, 0.012), (0.020, 0.012)]):
    cfg = lsgd.TrainConfig(algorithm=alg, n_workers=4, n_groups=G, layer_sizes=[16, 8, 4], n_samples=512,
                           n_features=16, n_classes=4, spread=6.0, local_batch=8, iterations=8, io_delay_s=io,
                           global_link_delay_s=link)
    cfg.b200.n_devices = nd
    cfg.b200.record_phases = rec
    r = lsgd.run_train(cfg)
    print(f"{alg} rec={int(rec)} io={io} link={link}: {1e3 * r.total_wall_s / 8:.2f} ms/block", flush=True)
