"""Debug: a 2-rank world where rank 1 never steps, on the NCCL paths (global_allreduce=nccl, flat CSGD). Prints what
rank 0 sees; each rank dumps its Python stack if it is still running after 60 s."""
import faulthandler
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def worker(rank, world, port, variant):
    faulthandler.dump_traceback_later(60, exit=True)
    import torch
    import torch.distributed as dist
    import paper_1906_05936_b200 as lsgd
    from paper_1906_05936_b200.executors import Rank
    from test_gpu_ranks import FLAT, _apply, _cfg
    torch.cuda.set_device(rank)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    over = FLAT if variant == "flat" else {"b200.global_allreduce": "nccl"}
    cfg = _apply(_cfg("fp64", world, 1 if variant == "flat" else 2), over)
    cfg.collective_timeout_s = 2.0
    r = Rank(cfg, rank, rank)
    blobs = [None] * world
    dist.all_gather_object(blobs, r.export())
    r.connect(blobs)
    r.synchronize()
    print(f"[{variant} r{rank}] connected", flush=True)
    if rank == 0:
        t0 = time.time()
        try:
            r.step(1)
            print(f"[{variant} r0] step issued {time.time() - t0:.1f}s", flush=True)
            r.synchronize()
            print(f"[{variant} r0] NO ERROR after {time.time() - t0:.1f}s", flush=True)
        except lsgd.LsgdError as e:
            print(f"[{variant} r0] {type(e).__name__}: {e} after {time.time() - t0:.1f}s", flush=True)
    dist.barrier()
    print(f"[{variant} r{rank}] closing", flush=True)
    r.close()
    print(f"[{variant} r{rank}] closed", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    from test_gpu_ranks import _free_port
    for variant in sys.argv[1:] or ["global", "flat"]:
        mp.spawn(worker, args=(2, _free_port(), variant), nprocs=2, join=True)
