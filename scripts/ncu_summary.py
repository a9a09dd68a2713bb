#!/usr/bin/env python
"""Summarise ncu output into profiles/ (run here, on the CPU box).

  ncu_summary.py full  <report.ncu-rep> <out.json> [--kernel REGEX]
  ncu_summary.py launches <launches.csv> <out.json>

`full` extracts the roofline counters of one `ncu --set full` capture (DRAM
bytes per launch, throughput percentages, occupancy, issue activity, stall
breakdown); `launches` aggregates a `--metrics gpu__time_duration.sum` launch
list into per-kernel counts, mean duration and share of the total.
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__shared_mem_per_block_dynamic",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__cycles_elapsed.avg", "gpc__cycles_elapsed.max", "dram__cycles_elapsed.avg.per_second",
]

UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0}


def full(rep, out, kernel=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kn = hdr.index("Kernel Name")
    res = []
    for r in data:
        if kernel and not re.search(kernel, r[kn]):
            continue
        d = {"kernel": r[kn]}
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[m] = v
                d[m + ".unit"] = units[i]
        stalls = {}
        for i, n in enumerate(hdr):
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v > 0.05:
                    stalls[n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        rb = d.get("dram__bytes_read.sum", 0) * UNIT.get(d.get("dram__bytes_read.sum.unit", "byte"), 1)
        wb = d.get("dram__bytes_write.sum", 0) * UNIT.get(d.get("dram__bytes_write.sum.unit", "byte"), 1)
        t = d.get("gpu__time_duration.sum", 0) * UNIT.get(d.get("gpu__time_duration.sum.unit", "ns"), 1e-9)
        d["dram_bytes_per_launch"] = rb + wb
        d["dram_gbs"] = (rb + wb) / t / 1e9 if t else None
        res.append(d)
    summary = {"report": rep, "launches": res}
    if res:
        summary["dram_bytes_per_launch"] = sum(x["dram_bytes_per_launch"] for x in res) / len(res)
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "launches"}))


def launches(path, out):
    text = open(path).read()
    start = text.index('"ID"') if '"ID"' in text else 0
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr, data = rows[0], rows[1:]
    kn, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in data:
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-9)
        agg[re.sub(r"\(.*", "", r[kn])].append(v)
    tot = sum(sum(v) for v in agg.values())
    res = {k: {"launches": len(v), "mean_ms": 1e3 * sum(v) / len(v), "total_ms": 1e3 * sum(v),
               "share": sum(v) / tot} for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}
    with open(out, "w") as f:
        json.dump({"source": path, "note": "ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, "
                   "serialised per-launch times; compare shares, not absolutes", "kernels": res}, f, indent=1)
    for k, v in res.items():
        print(f"{v['launches']:5d} {v['mean_ms']:10.4f} ms  {100 * v['share']:5.1f}%  {k}")


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        kern = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else None
        full(sys.argv[2], sys.argv[3], kern)
    else:
        launches(sys.argv[2], sys.argv[3])
