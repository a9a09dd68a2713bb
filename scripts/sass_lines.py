"""Attribute ncu per-SASS-instruction stall samples to CUDA source lines.

  sass_lines.py <ncu source csv (--print-source sass)> <nvdisasm -g -c dump> <function symbol>
"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) > 3]
iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
base = int(data[0][0], 16)
samples = {int(r[0], 16) - base: (float(r[iS] or 0), float(r[iE] or 0)) for r in data}

lines, cur, infn = {}, None, False
for l in open(sys.argv[2]):
    if l.startswith(".text."):
        infn = l.strip().rstrip(":") == ".text." + sys.argv[3]
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        lines[int(m.group(1), 16)] = cur
agg = defaultdict(lambda: [0.0, 0.0])
for off, (s, e) in samples.items():
    k = lines.get(off, "?")
    agg[k][0] += s
    agg[k][1] += e
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for k, (s, e) in sorted(agg.items(), key=lambda x: -x[1][0])[:40]:
    print(f"{k:30s} {100 * s / tot:5.1f}%  inst {e:.0f}")
