"""Exchange kernels in isolation (lsgd_b200_test_exchange_kernel): device time and achieved NVLink / HBM GB/s of
each production exchange kernel at the cfg3 slot size, device 0 pushing to 1 or 3 peers. Run plainly for the
CUDA-event numbers, under ncu (one process, no cross-GPU flags, so kernel replay is safe) for the counters:

    python tools/exchange_probe.py [--len 16777216] [--ndev 2,4] [--reps 20]
    ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        --clock-control none --csv python tools/exchange_probe.py --reps 1
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KINDS = {0: "reduce_push (K6 owner sum + push)", 1: "copy_pairs (scatter, SM stores)",
         2: "global_update (K7+K8 own slot + push)", 3: "update (K8, local)", 4: "cudaMemcpyAsync peer (copy engine)",
         5: "global_update + NVLS multimem.st fan-out"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--len", type=int, default=1 << 24, help="slot elements (fp32); cfg3 2x2 bucket sub-slice = 16M")
    ap.add_argument("--ndev", default="2,4")
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--kinds", default="0,1,2,3,4")
    args = ap.parse_args()
    from paper_1906_05936_b200 import _native as N

    lib = N.get_lib()
    f = lib.lsgd_b200_test_exchange_kernel
    f.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.POINTER(C.c_double),
                  C.POINTER(C.c_double), C.POINTER(C.c_double)]
    f.restype = C.c_int
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs") or 6650.0
    from paper_1906_05936_b200 import host
    ndev_max = host.device_count()
    for nd in [int(x) for x in args.ndev.split(",")]:
        if nd > ndev_max:
            continue
        for kind in [int(x) for x in args.kinds.split(",")]:
            ms, nv, loc = C.c_double(), C.c_double(), C.c_double()
            N.check(f(kind, nd, args.k, args.len, args.reps, C.byref(ms), C.byref(nv), C.byref(loc)))
            s = ms.value / 1e3
            print(json.dumps({"kernel": KINDS[kind], "kind": kind, "n_dev": nd, "k": args.k, "len": args.len,
                              "avg_ms": ms.value, "nvlink_bytes": nv.value, "hbm_bytes": loc.value,
                              "nvlink_gbs": nv.value / s / 1e9 if nv.value else None,
                              "nvlink_frac_of_770": nv.value / s / 770e9 if nv.value else None,
                              "hbm_gbs": loc.value / s / 1e9, "hbm_frac": loc.value / s / 1e9 / hbm}), flush=True)


if __name__ == "__main__":
    main()
