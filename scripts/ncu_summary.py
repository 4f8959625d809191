#!/usr/bin/env python
"""Summarise ncu output for profiles/: launch-list shares and per-kernel key counters.

    python scripts/ncu_summary.py launches gpurun_out/launches.csv
    python scripts/ncu_summary.py full gpurun_out/attn_full.ncu-rep [flops_per_launch ...]
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
              "second": 1e6, "s": 1e6}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    ours = {k: v for k, v in agg.items() if any(s in k for s in ("apb", "attn::", "score::", "sel::", "layer::", "dec::", "gemm::"))}
    tot = sum(v for _, v in agg.values())
    tot_ours = sum(v for _, v in ours.values())
    print(f"# ncu launch list ({path}); gpu__time_duration.sum, --clock-control none, serialised + cold-cache")
    print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'avg us':>10s} {'share all':>9s} {'share libapb':>12s}")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        s2 = f"{v / tot_ours * 100:11.1f}%" if k in ours else f"{'-':>12s}"
        print(f"{k[:70]:70s} {n:8d} {v / 1e3:10.3f} {v / n:10.1f} {v / tot * 100:8.1f}% {s2}")


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
]


def full(path, flops):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    name_i = h.index("Kernel Name")
    print(f"# ncu --set full summary of {path}")
    for n, r in enumerate(data):
        print(f"\n## launch {n}: {r[name_i][:110]}")
        vals = {}
        for w in WANT:
            if w in h:
                i = h.index(w)
                vals[w] = (r[i], units[i])
                print(f"  {w:70s} {r[i]:>16s} {units[i]}")
        if n < len(flops) and flops[n] > 0 and "gpu__time_duration.sum" in vals:
            t, u = vals["gpu__time_duration.sum"]
            t = float(t.replace(",", "")) * {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9}.get(u, 1.0)
            print(f"  {'useful TFLOP/s (mask-counted FLOPs / ncu duration)':70s} {flops[n] / t / 1e12:16.1f}")
        rd = vals.get("dram__bytes_read.sum")
        wr = vals.get("dram__bytes_write.sum")
        if rd and wr:
            sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = float(rd[0].replace(",", "")) * sc.get(rd[1], 1) + float(wr[0].replace(",", "")) * sc.get(wr[1], 1)
            print(f"  {'dram traffic (read+write) bytes':70s} {tot:16.0f}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], [float(x) for x in sys.argv[3:]])
