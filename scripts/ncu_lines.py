"""Per-source-line totals (instructions executed, stall samples) of the first
kernel in an ncu report: ncu -i REP --page source --csv --print-source cuda,sass
> file; python scripts/ncu_lines.py file [top]."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file, hdr, agg, fn_seen, first_fn = None, None, [], 0, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":  # one row per source file; stop at the next kernel
        if fn_seen and r[1] != first_fn:
            fn_seen = 2
        else:
            fn_seen, first_fn = 1, r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if fn_seen > 1:
        break
    if hdr and r[0]:
        iE = hdr.index("Instructions Executed")
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            agg.append((cur_file, int(r[0]), r[1][:70], float(r[iE] or 0), float(r[iS] or 0)))
        except ValueError:
            pass
tot_e = sum(a[3] for a in agg)
tot_s = sum(a[4] for a in agg)
print(f"total warp instructions {tot_e:.4g}, stall samples {tot_s:.4g}")
for f, ln, src, e, s in sorted(agg, key=lambda a: -a[3])[:top]:
    print(f"{f:22s}:{ln:4d} {100 * e / tot_e:5.1f}% inst {100 * s / tot_s:5.1f}% stall | {src}")
