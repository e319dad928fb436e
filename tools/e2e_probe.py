"""Probe of the end-to-end (host rows) path: PCIe H2D bandwidth, host enqueue time per step, device time per step."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_1906_05936_b200.executors import Rank

    torch.cuda.set_device(0)
    n = 8390656 // 4
    src = torch.empty(n, dtype=torch.float32).pin_memory()
    dst = torch.empty(n, dtype=torch.float32, device="cuda")
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"torch pinned H2D 8.4 MB: {ms * 1e3:.1f} us = {4 * n / ms / 1e6:.1f} GB/s; is_pinned={src.is_pinned()}")

    cfg = bench.workload("cfg3", 1, None, "lsgd")
    r = Rank(cfg, 0, 0)
    r.connect([r.export()])
    B, d, K = cfg.local_batch, cfg.n_features, 40
    xs = torch.randn((K, B, d), dtype=torch.float32).pin_memory()
    ys = torch.randint(0, cfg.n_classes, (K, B), dtype=torch.int32).pin_memory()
    lossbuf = torch.zeros(K, dtype=torch.float64, pin_memory=True)
    print("xs pinned", xs.is_pinned(), "ys pinned", ys.is_pinned())
    for t in range(5):
        r.step_rows(xs[t].data_ptr(), ys[t].data_ptr(), 1)
        r.loss_async(lossbuf.data_ptr() + 8 * t)
    r.synchronize()
    stream = torch.cuda.ExternalStream(r.stream())
    host = []
    e0.record(stream)
    t0 = time.perf_counter()
    for t in range(5, K):
        a = time.perf_counter()
        r.step_rows(xs[t].data_ptr(), ys[t].data_ptr(), 1)
        b = time.perf_counter()
        r.loss_async(lossbuf.data_ptr() + 8 * t)
        host.append((b - a, time.perf_counter() - b))
    r.join()
    e1.record(stream)
    t1 = time.perf_counter()
    r.synchronize()
    dev = e0.elapsed_time(e1) / (K - 5)
    hs = sorted(h[0] for h in host)
    print(f"rows path: device {dev:.3f} ms/step; host enqueue loop {(t1 - t0) * 1e3 / (K - 5):.3f} ms/step; "
          f"step_rows median {hs[len(hs) // 2] * 1e3:.3f} ms max {hs[-1] * 1e3:.3f} ms; loss_async median "
          f"{sorted(h[1] for h in host)[len(host) // 2] * 1e3:.3f} ms")
    e0.record(stream)
    r.step(K - 5)
    r.join()
    e1.record(stream)
    r.synchronize()
    print(f"index path: device {e0.elapsed_time(e1) / (K - 5):.3f} ms/step")
    r.close()


if __name__ == "__main__":
    main()
