"""BASELINE cfg5: gradient-size sweep of the LSGD exchange (reduce, global average, broadcast, update) at 2/4/8 GPUs.

    python sweep.py --gpus N [--groups G] [--sizes 20,22,24,26,28,30] [--steps 20] [--warmup 5]
    (spawns one process per GPU like bench.py; or torchrun --nproc-per-node N sweep.py ...)

Model = synthetic gradient (BASELINE cfg4/cfg5: g_r = Rng(1000 + r).next_symmetric(1.0), fp32), so a step is
exactly the communication path: postponed update (K8) -> intra-group ordered reduce (K6) -> inter-group NCCL average
(K7) -> push broadcast. Every kernel family is timed with CUDA events on its own stream (device time, max over
ranks). Reported per size, one JSON line on rank 0:
  reduce : per-GPU NVLink ingress (k-1)/k * 4P bytes (the sliced ordered reduce reads k-1 remote sub-slices)
  push   : per-GPU NVLink egress (k-1)/k * 4P bytes (each slot writes its averaged sub-slice to k-1 peers)
  global : NCCL allreduce of the 4P/k slice over G ranks, bus bytes 2(G-1)/G * 4P/k
  update : local HBM bytes 20P (momentum: read g, w, v; write w, v)
against the measured NVLink peer bandwidth (B200_PROFILING.md: 770 GB/s per direction) and MEASURED_PEAKS hbm_gbs.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", type=int, default=0, help="G (default: 1 for N<=2 else 2)")
    ap.add_argument("--sizes", default="20,22,24,26,28,30", help="log2 of P")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--global-allreduce", default="ordered", choices=["ordered", "nccl"])
    ap.add_argument("--gpus", type=int, default=0, help="spawn this many ranks (one per GPU) when not under torchrun")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import bench

        return bench.self_launch(sys.argv[1:], args.gpus, script=__file__)

    import torch
    import torch.distributed as dist

    import paper_1906_05936_b200 as lsgd
    from paper_1906_05936_b200.executors import Rank

    rank, local, world = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("LOCAL_RANK", 0), ("WORLD_SIZE", 1)))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    G = args.groups or (1 if world <= 2 else 2)
    k = world // G
    hbm = 6551.4
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, ValueError, KeyError):
        pass

    def gather(obj):
        if world == 1:
            return [obj]
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    for lg in (int(s) for s in args.sizes.split(",")):
        P = 1 << lg
        cfg = lsgd.TrainConfig(algorithm="lsgd", n_workers=world, n_groups=G, local_batch=1, n_samples=4096,
                               iterations=1 << 30, mode="momentum", layer_sizes=[32, 16, 10])
        cfg.b200.model = "synthetic_gradient"
        cfg.b200.synthetic_params = P
        cfg.b200.global_allreduce = args.global_allreduce
        r = Rank(cfg, rank, local)
        r.connect(gather(r.export()))
        r.step(args.warmup)
        r.synchronize()
        if world > 1:
            dist.barrier()
        r.timing(True)
        r.step(args.steps)
        r.synchronize()
        fam = {f: r.kernel_time(f) for f in ("scatter", "reduce", "global", "broadcast", "update")}
        r.timing(False)
        per_step = {f: (ms * cnt / args.steps) for f, (ms, cnt) in fam.items()}
        all_ps = gather(per_step)
        worst = {f: max(p[f] for p in all_ps) for f in per_step}
        r.close()
        if rank == 0:
            S = 4.0 * P / k
            line = {"metric": "LSGD exchange GB/s", "P": P, "n_gpus": world, "layout": f"{G}x{k}",
                    "ms_per_step": worst}

            def gbs(nbytes, ms):
                return nbytes / (ms * 1e-3) / 1e9 if ms > 0 else None

            line["scatter_nvlink_gbs"] = gbs((k - 1) * S, worst["scatter"]) if k > 1 else None
            line["reduce_push_gbs"] = gbs((G - 1) * S, worst["reduce"]) if G > 1 else None
            line["push_nvlink_gbs"] = gbs((k - 1) * S, worst["broadcast"]) if k > 1 else None
            sliced = G > 2 or (G > 1 and k == 1)  # the engine's default (rank.cu sliced_global)
            if args.global_allreduce == "nccl":
                line["global_busbw_gbs"] = gbs(2 * (G - 1) / G * S, worst["global"]) if G > 1 else None
            else:  # fused global kernel: ordered group sum + update of the own slot (piece) + fan-out of its average
                line["global_push_gbs"] = gbs((world - 1) * S / G if sliced else (k - 1) * S, worst["global"])
            line["global_allreduce"] = args.global_allreduce
            # the update kernel covers the slots (pieces) this GPU does not own: 20 B per parameter (momentum)
            own = (1.0 / world if sliced else 1.0 / k) if world > 1 else 0.0
            line["update_hbm_gbs"] = gbs(20.0 * P * (1.0 - own), worst["update"])
            line["nvlink_peak_gbs"] = NVLINK_GBS
            line["hbm_peak_gbs"] = hbm
            print(json.dumps(line), flush=True)
        if world > 1:
            dist.barrier()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
