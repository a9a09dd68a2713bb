"""Warp instructions per launch of each C2 scoring-model variant, from the ncu
launch list of scripts/model_variants_prof.py (2 launches per variant, in
bench.model_variant_specs order; the second is kept) -> profiles/model_variants_instr.json."""
import csv
import json
import sys

VARIANTS = ["eq3/edge/1 step", "eq3/uniform/1 step", "eq3/edge/3 steps", "log_grid/uniform/3 steps"]
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h = rows[0]
iI, iK, iM, iV = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = {}
for r in rows[1:]:
    if r[iM] == "smsp__inst_executed.sum" and "prep" not in r[iK]:
        per[int(r[iI])] = (r[iK], float(r[iV].replace(",", "")))
ids = sorted(per)
assert len(ids) == 2 * len(VARIANTS), len(ids)
out = {"source": sys.argv[1], "kernels": {}, "instructions_per_launch": {}}
for j, name in enumerate(VARIANTS):
    k, v = per[ids[2 * j + 1]]
    out["instructions_per_launch"][name] = int(v)
    out["kernels"][name] = k
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
