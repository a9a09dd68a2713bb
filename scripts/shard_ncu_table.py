"""Summarise the launch lists of scripts/gpu_shard_ncu.sh: per launch (second
rep of each family) time, warp instructions, warps active, issue active."""
import csv
import sys

for fn in sys.argv[1:]:
    rows = [r for r in csv.reader(l for l in open(fn) if l.startswith('"'))]
    h = rows[0]
    iI, iK, iM, iV = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = {}
    for r in rows[1:]:
        per.setdefault(int(r[iI]), {"k": r[iK].split("(")[0].replace("void ", "")})[r[iM]] = float(r[iV].replace(",", ""))
    ids = sorted(per)
    tot_t = tot_i = 0
    print(fn)
    for i in ids:
        if (i // 2) % 2 == 0:      # first rep of each family (2 launches per rep, 2 reps per family)
            continue
        d = per[i]
        tot_t += d["gpu__time_duration.sum"]
        tot_i += d["smsp__inst_executed.sum"]
        print(f"  {d['k']:32s} {d['gpu__time_duration.sum']/1e3:9.1f} us {d['smsp__inst_executed.sum']/1e9:7.3f} G  "
              f"warps {d['sm__warps_active.avg.pct_of_peak_sustained_active']:5.1f}%  "
              f"issue {d['smsp__issue_active.avg.pct_of_peak_sustained_active']:5.1f}%")
    print(f"  total {tot_t/1e3:.1f} us serialised, {tot_i/1e9:.3f} G warp instructions")
