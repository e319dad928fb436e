"""CPU, world_size = 2 over gloo (127.0.0.1): the host-side logic every rank of a one-process-per-GPU world runs
before its GPU work — shard of the global minibatch, topology, learning-rate schedule, rank bootstrap — agrees across
ranks and with the oracle (sampler.cpp:45-57, executors.cpp:389-433), and the rank API fails loudly without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import paper_1906_05936_b200 as lsgd
    from paper_1906_05936_b200 import host

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=world * 2, n_groups=2, layer_sizes=[16, 8, 4],
                               n_samples=300, n_features=16, n_classes=4, spread=6.0, local_batch=8, iterations=40)
        # each process owns workers [2*rank, 2*rank+2) (two GPUs' worth of shards per process)
        idx = host.minibatch_indices(cfg, 0, 5)
        mine = idx[:, rank * 2 * cfg.local_batch:(rank + 1) * 2 * cfg.local_batch]
        gathered = [None] * world
        dist.all_gather_object(gathered, (mine.tolist(), host.topology(cfg), host.learning_rate(cfg, 17)))
        err = None
        try:
            r = lsgd.executors.Rank(cfg, rank, 0)  # no GPU in this container: must fail, loudly, not fall back
            r.close()
        except lsgd.LsgdError as e:
            err = type(e).__name__
        if rank == 0:
            out["gathered"] = gathered
            out["idx"] = idx.tolist()
            out["err"] = err
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_world_agrees_on_host_state():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    idx = np.array(out["idx"])
    shards = [np.array(g[0]) for g in out["gathered"]]
    # the two processes' shards tile the global minibatch in worker order
    assert np.array_equal(np.concatenate(shards, axis=1), idx)
    # topology and the LR schedule are identical on every rank
    t0, t1 = out["gathered"][0][1], out["gathered"][1][1]
    assert all(np.array_equal(np.asarray(a), np.asarray(b)) for a, b in zip(t0, t1))
    assert out["gathered"][0][2] == out["gathered"][1][2]
    # and the minibatch stream is the oracle's: SplitMix64 Fisher-Yates draws of the global batch with the sampler
    # seed (seed + 2, sampler.cpp:15-43), partitioned contiguously over the workers (:45-57)
    from oracle import Oracle
    o = Oracle("port")
    draws, _ = o.sampler(300, 42 + 2, 4 * 8, 5)
    for t in range(5):
        assert np.array_equal(o.partition(draws[t], 4).reshape(-1), idx[t])
    assert out["err"] is not None, "Rank creation without a GPU must raise"
