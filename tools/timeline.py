"""Device timeline of a few cfg3 steps (CUDA events per launch family, all streams), for schedule tuning.

    python tools/timeline.py [--workload cfg3] [--algo lsgd] [--steps 3]      (one GPU)
    torchrun --nproc-per-node N tools/timeline.py ...                        (rank 0 prints)
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--algo", default="lsgd")
    ap.add_argument("--global-allreduce", default="ordered")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--rows", action="store_true", help="e2e path: pinned host rows (step_rows) + async loss D2H")
    ap.add_argument("--all-ranks", action="store_true", help="also write gpurun_out/timeline_rank<r>.txt per rank")
    ap.add_argument("--groups", type=int, default=None)
    args = ap.parse_args()
    import torch

    import bench
    from paper_1906_05936_b200 import _native as N
    from paper_1906_05936_b200.executors import Rank

    rank, local, world = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("LOCAL_RANK", 0), ("WORLD_SIZE", 1)))
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        pg = dist

    def allgather(o):
        if not pg:
            return [o]
        out = [None] * world
        pg.all_gather_object(out, o)
        return out

    cfg = bench.workload(args.workload, world, None, args.algo, args.global_allreduce, args.groups)
    r = Rank(cfg, rank, local)
    if rank == 0:
        print("# buckets (id: layer rows n):", ", ".join(f"{i}: L{b[0]} {b[1]} {b[2]}" for i, b in enumerate(r.buckets()))
              if hasattr(r, "buckets") else "")
    r.connect(allgather(r.export()))
    if args.rows:
        B, d = cfg.local_batch, cfg.n_features
        K = args.warmup + args.steps
        xs = torch.randn((K, B, d), dtype=torch.float32).pin_memory()
        ys = torch.randint(0, cfg.n_classes, (K, B), dtype=torch.int32).pin_memory()
        lossbuf = torch.zeros(K, dtype=torch.float64, pin_memory=True)

        def run(t0, n):
            for t in range(t0, t0 + n):
                r.step_rows(xs[t].data_ptr(), ys[t].data_ptr(), 1)
                r.loss_async(lossbuf.data_ptr() + 8 * t)
    else:
        def run(t0, n):
            r.step(n)
    run(0, args.warmup)
    r.synchronize()
    if pg:
        pg.barrier()
    r.timing(True)
    run(args.warmup, args.steps)
    r.join()
    r.synchronize()
    fn = N.lib.lsgd_b200_test_rank_timeline
    fn.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
    fn.restype = C.c_int
    buf = C.create_string_buffer(1 << 20)
    N.check(fn(r.h, buf, len(buf)))
    lines = [ln.split("\t") for ln in buf.value.decode().strip().splitlines()]
    if args.all_ranks:  # every rank's timeline (origin: each rank's timing(True) right after a host barrier)
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"timeline_rank{rank}.txt"), "w") as f:
            for fam, a, b, tag in lines:
                f.write(f"{fam:10s} {tag:>4s} {float(a):9.3f} {float(b):9.3f} {1e3 * (float(b) - float(a)):8.1f} us\n")
    if rank == 0:
        tot = {}
        for fam, a, b, tag in lines:  # tag: bucket id, 100 + k forward / 200 + k dX GEMM of layer k
            tot[fam] = tot.get(fam, 0.0) + float(b) - float(a)
            print(f"{fam:10s} {tag:>4s} {float(a):9.3f} {float(b):9.3f} {1e3 * (float(b) - float(a)):8.1f} us")
        end = max(float(b) for _, b in ((ln[1], ln[2]) for ln in lines))
        print(f"# {args.steps} steps span {end:.3f} ms ({end / args.steps:.3f} ms/step); busy ms per family: "
              + ", ".join(f"{k}={v / args.steps:.3f}" for k, v in sorted(tot.items())))
    r.close()
    if pg:
        pg.barrier()
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
