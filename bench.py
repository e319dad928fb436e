"""Benchmark of the LSGD synchronous update step (BASELINE.json metric: samples/sec at 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--workload cfg3|cfg1|cfg4]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU; driver-launched for N > 1)

Default workload (N=1 and the scaling run): BASELINE cfg3 — wide MLP 4096-8192-8192-512 (P = 104,874,496 fp32),
synthetic Gaussian blobs (n = 65,536), B_loc = 512 samples per GPU (weak scaling), layout G x k with
G = min(2, N) communicator groups (N=8 -> 2 x 4 as BASELINE cfg3 names), momentum SGD. A step = io (shard index
H2D + row gather), postponed broadcast+update of the previous round, forward/backward, ordered intra-group
reduce, inter-group NCCL average on the side stream.

`value`  : samples/s over K steps with the dataset resident in HBM, device-timed (CUDA events on the rank's
           stream), max over ranks.
`e2e`    : the same metric through the C-ABI data-loader call with HOST buffers: each step's shard rows are
           copied H2D from pinned memory and the round's loss is read back D2H inside the timed region.
`roofline`: the dominant kernel family (the tensor-core GEMM sequence of forward+backward) against the measured
           dense-GEMM peak in MEASURED_PEAKS.json; the reduce/update kernels are reported in `kernels`.
`cpu_baseline`: the reference's own run_train (oracle/_ref, built from /root/reference sources) on the host cores.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec (LSGD step, weak scaling, B_loc per GPU)"
UNIT = "samples/s"


def workload(name: str, n: int, bloc: int | None, algo: str, glob: str = "ordered", groups: int | None = None):
    import paper_1906_05936_b200 as lsgd

    G = (groups or min(2, n)) if algo == "lsgd" else 1
    if n % G:
        raise SystemExit(f"--groups {G} does not divide {n} workers")
    if name == "cfg3":
        layers = [4096, 8192, 8192, 512]
        cfg = lsgd.TrainConfig(algorithm=algo, n_workers=n, n_groups=G, layer_sizes=layers, n_samples=65536,
                               n_features=4096, n_classes=512, spread=10.0, mode="momentum",
                               local_batch=bloc or 512, iterations=1 << 30, seed=42)
    elif name == "cfg1":
        cfg = lsgd.TrainConfig(algorithm=algo, n_workers=n, n_groups=G, layer_sizes=[32, 16, 10], n_samples=5000,
                               n_features=32, n_classes=10, spread=10.0, mode="momentum",
                               local_batch=bloc or 16, iterations=1 << 30, seed=42)
    elif name == "cfg4":
        cfg = lsgd.TrainConfig(algorithm=algo, n_workers=n, n_groups=G, layer_sizes=[32, 16, 10], n_samples=5000,
                               mode="momentum", local_batch=bloc or 64, iterations=1 << 30, seed=42)
        cfg.b200.model = "synthetic_gradient"
        cfg.b200.synthetic_params = 25_600_000
    else:
        raise SystemExit(f"unknown workload {name}")
    cfg.b200.global_allreduce = glob
    if algo == "csgd":
        cfg.b200.csgd_nccl = True
    return cfg


def flops_per_sample(layers):
    """F = 2*sum in*out (fwd) + 2*sum in*out (dW) + 2*sum_{k>=1} in*out (dX; layer 0 skipped, mlp.cpp:116)."""
    f = sum(2 * layers[k] * layers[k + 1] for k in range(len(layers) - 1))
    return 2 * f + sum(2 * layers[k] * layers[k + 1] for k in range(1, len(layers) - 1))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.stop = gpu, [], threading.Event()
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def finish(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for i, nm in enumerate(names):
                    if r[5 + i].lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ------------------------------------------------------------------------------------------------ reference arm
def cpu_reference(cfg_name: str, n: int, steps: int, warmup: int, bloc: int | None, algo: str,
                  groups: int | None = None):
    """The reference's own run_train (UNMODIFIED sources, oracle/_ref) timed on the host cores."""
    from oracle import Oracle, TrainSpec

    cores = os.cpu_count() or 1
    # every host thread the box has: each of the n worker ranks gets cores / n OpenMP threads for its per-sample
    # passes (batch_gradient parallelises over the samples of a 32-sample block, mlp.cpp:249-257), and B_loc matches
    # that thread count so none idles. libgomp reads OMP_NUM_THREADS when the reference library loads.
    os.environ.setdefault("OMP_NUM_THREADS", str(max(1, cores // max(1, n))))
    ref = Oracle("reference")
    if cfg_name == "cfg3":
        # OpenMP gradient scratch is min(32, B) x P doubles (mlp.cpp:243-245): keep B_loc small, dataset small
        # bounded sample (~10-60 s of CPU work whatever --steps is): a few iterations at a small per-worker batch;
        # the reference's per-sample cost does not depend on the batch or dataset size
        b = max(1, min(32, cores // max(1, n)))
        iters = max(1, min(steps, 3))
        spec = TrainSpec(algorithm=algo, n_workers=n, n_groups=(groups or min(2, n)) if algo == "lsgd" else 1,
                         layer_sizes=[4096, 8192, 8192, 512], n_samples=max(1024, 4 * b * n), n_features=4096,
                         n_classes=512, mode="momentum", local_batch=b, iterations=iters)
        sample = (f"run_train lsgd {spec.n_groups}x{n // spec.n_groups}, MLP 4096-8192-8192-512 fp64, B_loc={b}, "
                  f"{iters} iterations on {spec.n_samples} blobs (per-step cost is independent of n)")
    else:
        b = bloc or 16
        spec = TrainSpec(algorithm=algo, n_workers=n, n_groups=(groups or min(2, n)) if algo == "lsgd" else 1,
                         layer_sizes=[32, 16, 10], mode="momentum", local_batch=b, iterations=max(steps, 100))
        sample = f"run_train {algo} N={n}, MLP 32-16-10 fp64, B_loc={b}, {spec.iterations} iterations"
    if warmup:
        w = TrainSpec(**{**spec.__dict__, "iterations": 1})
        ref.run_train(w)
    out = ref.run_train(spec)
    return {"value": out["throughput_sps"], "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample,
            "omp_threads": int(os.environ["OMP_NUM_THREADS"]), "rank_threads": spec.n_workers + spec.n_groups}


def run_reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    cb = cpu_reference(args.workload, args.gpus, args.steps, args.warmup, args.bloc, args.algo, args.groups)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload} on host cores (reference CPU implementation)",
                       "algorithm": args.algo},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------ b200 arm
def run_b200_arm(args):
    import numpy as np
    import torch

    from paper_1906_05936_b200.executors import Rank

    rank, local, world = dist_env()
    n = world if world > 1 else args.gpus
    if world == 1 and args.gpus > 1:
        raise SystemExit("--gpus > 1 needs one process per GPU (bench.py self-launches them when WORLD_SIZE is "
                         "unset; this rank saw WORLD_SIZE=1)")
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
        pg = dist

    def barrier():
        if pg:
            pg.barrier()

    def allgather(obj):
        if not pg:
            return [obj]
        out = [None] * world
        pg.all_gather_object(out, obj)
        return out

    cfg = workload(args.workload, n, args.bloc, args.algo, args.global_allreduce, args.groups)
    t_setup = time.time()
    print(f"[bench rank {rank}/{world}] creating Rank on device {local}", file=sys.stderr, flush=True)
    r = Rank(cfg, rank, local)  # fails loudly (LsgdError / ImportError) without an sm_100 GPU or the library
    torch.cuda.set_device(local)
    r.connect(allgather(r.export()))
    r.synchronize()
    setup_s = time.time() - t_setup
    stream = torch.cuda.ExternalStream(r.stream())

    # warm-up, then K timed steps bracketed by barrier + sync (max over ranks)
    r.step(args.warmup)
    r.synchronize()
    barrier()
    r.timing(True)
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    l0 = r.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r.synchronize()
    barrier()
    ev0.record(stream)
    r.step(args.steps)
    r.join()  # the last step's update / exchange streams finish inside the timed region
    ev1.record(stream)
    r.synchronize()
    ms = ev0.elapsed_time(ev1)
    nvlink = None
    if n > 1:
        G_, k_ = cfg.n_groups, n // cfg.n_groups
        # algorithmic egress per GPU and step: scatter (k-1)S + group-sum push (G-1)S + average fan-out (k-1)S with
        # S = 4(P+1)/k (push exchange); flat allreduce 2(N-1)/N * 4(P+1). Achieved = over the step time (the
        # exchange overlaps the GEMMs); the kernels alone: profiles/r2_ncu_exchange_kernels.json
        tx = (4.0 * (cfg.n_params + 1) * (2 * k_ + G_ - 3) / k_ if args.algo == "lsgd"
              else 2.0 * (n - 1) / n * 4.0 * (cfg.n_params + 1))
        nvlink = {"algorithmic_tx_bytes_per_step": tx, "tx_gbs_over_step": tx / (ms / args.steps / 1e3) / 1e9,
                  "peak_gbs": 770.0, "peak_source": "B200_PROFILING.md measured peer copy per direction"}
    launches = r.launches() - l0
    clk = clocks.finish() if clocks else None
    r.timing(False)
    fams = {f: r.kernel_time(f) for f in ("gemm", "scatter", "reduce", "global", "broadcast", "update", "gather",
                                          "bias", "head", "split")}
    ms_all = allgather(ms)
    ms_max = max(ms_all)
    B = cfg.local_batch
    value = args.steps * n * B / (ms_max / 1e3)

    # t_step(1) for SURVEY.md §8(d)'s exposed communication (t_step(N) - t_step(1)): rank 0 runs the same workload
    # as one worker on its own GPU, same K / W, right after the N-GPU measurement (the other ranks wait)
    t1_ms = None
    if n > 1 and cfg.b200.model == "mlp" and not args.skip_t1:
        if rank == 0:
            c1 = workload(args.workload, 1, args.bloc, "lsgd", args.global_allreduce, 1)
            r1 = Rank(c1, 0, local)
            r1.connect([r1.export()])
            s1 = torch.cuda.ExternalStream(r1.stream())
            r1.step(args.warmup)
            r1.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s1)
            r1.step(args.steps)
            r1.join()
            e1.record(s1)
            r1.synchronize()
            t1_ms = e0.elapsed_time(e1) / args.steps
            r1.close()
            del r1
        barrier()

    # e2e: host rows -> H2D per step, loss D2H per step, through the C-ABI data-loader call
    e2e = None
    if cfg.b200.model == "mlp" and not args.skip_e2e:
        d = cfg.n_features
        from paper_1906_05936_b200 import host

        K, W = args.steps, args.warmup
        idx = host.minibatch_indices(cfg, 10_000, K + W)[:, rank * B:(rank + 1) * B]
        xs = torch.empty((K + W, B, d), dtype=torch.float32, pin_memory=True)
        ys = torch.empty((K + W, B), dtype=torch.int32, pin_memory=True)
        # host-side gather of the shard rows (the data loader's job) happens before the timed region
        xh, yh = host.generate_synthetic(cfg.seed, cfg.n_samples, d, cfg.n_classes, cfg.spread)
        xs.copy_(torch.from_numpy(xh[idx].astype(np.float32)))
        ys.copy_(torch.from_numpy(yh[idx].astype(np.int32)))
        del xh, yh
        lossbuf = torch.zeros(K + W, dtype=torch.float64, pin_memory=True)  # per-step D2H destination
        esz = 8

        def rows_steps(t0, n):
            nonlocal esz
            for t in range(t0, t0 + n):
                r.step_rows(xs[t].data_ptr(), ys[t].data_ptr(), 1)
                # D2H of the applied round's loss, ordered after its update; the host does not block, so the next
                # step's H2D (copy stream) overlaps this step's compute
                esz = r.loss_async(lossbuf.data_ptr() + 8 * t)

        rows_steps(0, W)  # warm-up of the host-rows path (staging buffers, copy stream)
        r.synchronize()
        barrier()
        t0 = time.perf_counter()
        ev0.record(stream)
        rows_steps(W, K)
        t_issue = time.perf_counter() - t0
        r.join()
        ev1.record(stream)
        r.synchronize()
        e2e_ms = max(allgather(ev0.elapsed_time(ev1)))
        raw = lossbuf.numpy().view(np.uint8).reshape(K + W, 8)[W:, :esz].copy()
        losses = raw.view(np.float32 if esz == 4 else np.float64).ravel()
        e2e = {"value": K * n * B / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": B * d * 4 + B * 4,
               "d2h_bytes_per_step": esz, "wall_s": time.perf_counter() - t0, "host_issue_s": t_issue,
               "loss_finite": bool(np.all(np.isfinite(losses))), "loss_last": float(losses[-1])}

    # CPU baseline (rank 0, N=1 only): the reference itself on the host cores, bounded sample
    cpu = None
    if rank == 0 and n == 1 and not args.skip_cpu:
        try:
            cpu = cpu_reference(args.workload, 1, 3, 0, args.bloc, args.algo)
        except Exception as e:  # reference build missing on this box
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        peaks = measured_peaks()
        roof = None
        if cfg.b200.model == "mlp":
            F = flops_per_sample(cfg.layer_sizes)
            avg, cnt = fams["gemm"]
            gemm_n = cnt
            gemm_ms = avg * cnt / args.steps  # per-layer brackets summed to one step's GEMM time
            ach = (B * F) / (gemm_ms / 1e3) / 1e12 if gemm_ms else None
            peak = peaks.get("bf16_tflops_sustained") or 1400.0
            traffic, tsrc = None, None
            for cand in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_gemm.json")), reverse=True):
                try:  # DRAM bytes of one step's GEMM sequence from the committed ncu --set full capture
                    traffic = json.load(open(cand))["step_gemm_dram_mb"] * 1e6
                    tsrc = os.path.relpath(cand, ROOT)
                    break
                except (OSError, ValueError, KeyError):
                    pass
            tf32 = None
            try:  # measured dense TF32 peak on a B200 of this pool (tools/tf32_peak.py)
                tf32 = json.load(open(os.path.join(ROOT, "profiles", "r2_tf32_peak.json")))["tf32_tflops_sustained"]
            except (OSError, ValueError, KeyError):
                pass
            roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                    "frac": (ach / peak) if ach else None, "traffic": traffic, "traffic_source": tsrc,
                    "traffic_unit": "bytes DRAM read+write per launch (= one step's GEMM sequence)",
                    "kernel": "forward+backward GEMM sequence per step (B_loc*F flops / its device time)",
                    "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (3xTF32 ceiling = peak/6)",
                    "frac_of_3xtf32_ceiling": (ach / (peak / 6)) if ach else None,
                    "tf32_tflops_measured": tf32,
                    "frac_of_measured_split_tf32_ceiling": (ach / (tf32 / 3)) if (ach and tf32) else None,
                    "split_tf32_note": "each fp32 product = 3 TF32 MMAs (hi*hi + hi*lo + lo*hi): ceiling = TF32 / 3; "
                                       "TF32 measured with cuBLAS (profiles/r2_tf32_peak.json)",
                    "flops_per_launch": B * F, "launches_timed": gemm_n}
        else:
            # synthetic gradient: the step is exchange + update; the roofline kernel is the update pass. With an
            # exchange the owner's own slot is updated inside the fused global kernel, so the update kernel covers
            # the (k-1)/k other slots; with one worker per group (k = 1) the fused global kernel does all of it.
            P = cfg.n_params
            G = cfg.n_groups
            k = n // G
            wv = 4 * (2 if cfg.mode == "momentum" else 1)  # w (+ v) bytes per parameter, each read and written
            if n > 1 and k == 1:
                fam, kname = "global", "K7+K8 global_update (ordered group sum + update, whole slot)"
                bytes_ = P * (4 * G + 2 * wv)  # own payload + G-1 group sums read, w (+ v) read + written
            else:
                fam, kname = "update", "K8 update (broadcast average + momentum update)"
                bytes_ = P * (4 + 2 * wv) * ((k - 1) / k if n > 1 else 1.0)  # average read, w (+ v) read + written
            avg, cnt = fams[fam]
            up_ms = avg * cnt / args.steps
            ach = bytes_ / (up_ms / 1e3) / 1e9 if up_ms else None
            peak = peaks.get("hbm_gbs") or 6650.0
            roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": (ach / peak) if ach else None,
                    "traffic": None, "kernel": kname, "bytes_per_launch_step": bytes_}
        # step-level roofline of the north star: t_roof = max(B_loc*F / GEMM_peak,
        # 4(P+1) / BW_NVLink), GEMM_peak = the 3xTF32 effective rate of the measured dense peak (peak/6)
        step_roof = None
        if cfg.b200.model == "mlp":
            gemm_peak = (peaks.get("bf16_tflops_sustained") or 1400.0) / 6.0 * 1e12
            t_gemm = B * flops_per_sample(cfg.layer_sizes) / gemm_peak
            t_link = 4.0 * (cfg.n_params + 1) / 900e9 if n > 1 else 0.0
            t_roof = max(t_gemm, t_link)
            step_roof = {"t_roof_ms": t_roof * 1e3, "t_step_ms": ms_max / args.steps,
                         "frac": t_roof * 1e3 / (ms_max / args.steps), "t_gemm_ms": t_gemm * 1e3,
                         "t_nvlink_ms": t_link * 1e3,
                         "basis": "SURVEY.md §8(d): 3xTF32 = bf16_tflops_sustained/6; 4(P+1) B over NVLink 900 GB/s"}
            # the same bound with the measured ceilings: split-TF32 = measured TF32 / 3, and the exchange's
            # algorithmic egress 2(N-1)/N * 4(P+1) B at the measured 770 GB/s peer bandwidth
            try:
                tf32 = json.load(open(os.path.join(ROOT, "profiles", "r2_tf32_peak.json")))["tf32_tflops_sustained"]
                t_g = B * flops_per_sample(cfg.layer_sizes) / (tf32 / 3.0 * 1e12)
                t_l = 2.0 * (n - 1) / n * 4.0 * (cfg.n_params + 1) / 770e9 if n > 1 else 0.0
                step_roof["measured"] = {"t_gemm_ms": t_g * 1e3, "t_nvlink_ms": t_l * 1e3,
                                         "frac": max(t_g, t_l) / (ms_max / args.steps / 1e3)}
            except (OSError, ValueError, KeyError):
                pass
        kern = {f: {"avg_ms": v[0], "count": v[1], "ms_per_step": v[0] * v[1] / args.steps}
                for f, v in fams.items() if v[1]}
        # exposed communication (BASELINE metric): step time not covered by the main stream's compute kernels
        # (rank 0's per-step device time of its GEMMs, gather, head, split; the bias gradients run on their own
        # stream under LSGD, on the main stream otherwise)
        exposed = None
        if cfg.b200.model == "mlp":
            main_fams = ["gemm", "gather", "head", "split"]
            if os.environ.get("LSGD_B200_BIAS_STREAM") == "0":
                main_fams.append("bias")
            main_ms = sum(kern[f]["ms_per_step"] for f in main_fams if f in kern)
            exposed = {"ms_per_step": (ms_max / args.steps - t1_ms) if t1_ms is not None else 0.0,
                       "t_step_n_ms": ms_max / args.steps, "t_step_1_ms": t1_ms if n > 1 else ms_max / args.steps,
                       "basis": "SURVEY.md §8(d): t_step(N) - t_step(1), t_step(1) = the same workload as one "
                                "worker on rank 0's GPU in the same run",
                       "beyond_main_compute_ms": max(0.0, ms_max / args.steps - main_ms),
                       "main_compute_ms": main_ms}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": args.workload, "model": "MLP " + "-".join(map(str, cfg.layer_sizes))
                           if cfg.b200.model == "mlp" else f"synthetic gradient P={cfg.n_params}",
                           "algorithm": args.algo, "layout": f"{cfg.n_groups}x{n // cfg.n_groups}",
                           "local_batch": B, "global_batch": B * n, "n_params": cfg.n_params,
                           "global_allreduce": cfg.b200.global_allreduce,
                           "l2": "working set (w, v, grad, slices) >> 126 MB L2; no flush needed"},
                "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clk,
                "step_roofline": step_roof, "exposed_comm": exposed, "nvlink": nvlink, "kernels": kern, "setup_s": setup_s}
        print(json.dumps(line), flush=True)
    r.close()
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def self_launch(argv, n, script=None):
    """`bench.py --gpus N` without torchrun: spawn N rank processes (one per GPU) on a 127.0.0.1 rendezvous, the
    environment torchrun would give them; rank 0's stdout is this process's stdout. Any rank failing stops the
    others and the job exits non-zero."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(script or __file__)] + argv, env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    try:
        while procs:
            for p in list(procs):
                c = p.poll()
                if c is None:
                    continue
                procs.remove(p)
                if c != 0:
                    rc = rc or c
                    for q in procs:  # the survivors would wait in a barrier forever
                        q.terminate()
            time.sleep(0.05)
    finally:
        for p in procs:
            p.kill()
    return rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=["cfg3", "cfg1", "cfg4"])
    ap.add_argument("--algo", default="lsgd", choices=["lsgd", "csgd"])
    ap.add_argument("--global-allreduce", default="ordered", choices=["nccl", "ordered"],
                    help="LSGD inter-group average: NCCL over the slot owners, or the ordered push sum")
    ap.add_argument("--bloc", type=int, default=None)
    ap.add_argument("--groups", type=int, default=None,
                    help="LSGD communicator groups (default min(2, N): N=8 -> 2x4); e.g. 1 for 1xN, N for Nx1")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-t1", action="store_true", help="skip the in-run t_step(1) of exposed_comm at N > 1")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(sys.argv[1:], args.gpus)
    return run_b200_arm(args)


if __name__ == "__main__":
    sys.exit(main())
