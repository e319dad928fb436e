"""Summarise the 1-GPU ncu captures of tools/profile_n1.sh into profiles/ (tracked).

    python tools/ncu_summary.py gpurun_out/prof_gemm.ncu-rep gpurun_out/launches.csv profiles/r1

Writes <prefix>_ncu_gemm.json (per GEMM launch: shape, duration, DRAM bytes, tensor-pipe / L2 / DRAM utilisation,
top stall reasons; totals per step = the roofline `traffic`) and <prefix>_launches.json (kernel time shares of the
serialised, cold-cache launch list of the bench command).
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

WANT = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_mb",
    "dram__bytes_write.sum": "dram_write_mb",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}
UNIT_SCALE = {"usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0,
              "Gbyte": 1e3}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, launches, prefix = sys.argv[1:4]
    hdr, units, rows = raw_rows(rep)
    col = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    gemms = []
    for r in rows:
        g = {"kernel": r[col["Kernel Name"]].split("(")[0].replace("void ", "")}
        for k, name in WANT.items():
            if k not in col:
                continue
            v = r[col[k]]
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            x *= UNIT_SCALE.get(units[col[k]], 1.0) if name.endswith(("_us", "_mb")) else 1.0
            g[name] = x
        st = sorted(((float(r[col[h]] or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h in stall_cols),
                    reverse=True)[:4]
        tot = sum(float(r[col[h]] or 0) for h in stall_cols) or 1.0
        g["top_stalls_pct"] = {n: round(100 * v / tot, 1) for v, n in st}
        gemms.append(g)
    tot_dram = sum(g.get("dram_read_mb", 0) + g.get("dram_write_mb", 0) for g in gemms)
    tot_us = sum(g.get("duration_us", 0) for g in gemms)
    summary = {"source": rep, "captured": "ncu --set full --clock-control none, one bench step's GEMM launches "
               "(serialised replays: per-launch times are cold-cache, use the shares, not the absolutes)",
               "launches": gemms, "step_gemm_dram_mb": tot_dram, "step_gemm_us_serialised": tot_us}
    with open(prefix + "_ncu_gemm.json", "w") as f:
        json.dump(summary, f, indent=1)
    # launch list: per-kernel time share
    per = defaultdict(lambda: [0.0, 0])
    with open(launches) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.reader(lines)
    h = next(rd)
    ci = {x: i for i, x in enumerate(h)}
    for r in rd:
        if r[ci["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ci["Kernel Name"]].split("(")[0].replace("void ", "")
        name = name.split("<")[0] if "ncclDevKernel" not in name else name
        v = float(r[ci["Metric Value"]].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(
            r[ci["Metric Unit"]], 1.0)
        per[name][0] += v * scale
        per[name][1] += 1
    total = sum(v[0] for v in per.values()) or 1.0
    share = {k: {"us": round(v[0], 1), "launches": v[1], "share_pct": round(100 * v[0] / total, 1)}
             for k, v in sorted(per.items(), key=lambda kv: -kv[1][0])}
    with open(prefix + "_launches.json", "w") as f:
        json.dump({"source": launches, "total_us": total, "kernels": share}, f, indent=1)
    print(json.dumps({"step_gemm_dram_mb": tot_dram, "step_gemm_us": tot_us,
                      "top": list(share.items())[:6]}, indent=1))


if __name__ == "__main__":
    main()
