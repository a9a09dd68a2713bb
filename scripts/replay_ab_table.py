"""Summarise gpurun_out/replay_ab.log (scripts/gpu_replay_ab.sh): sweep ms and shard-proxy max per N."""
import json
import sys

label = None
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/replay_ab.log"):
    if line.startswith("== "):
        label = line[3:].strip()
    elif line.startswith("{"):
        r = json.loads(line)["replay"]
        sp = r.get("shard_proxy", {})
        print(f"{label:10s} sweep {r['ms_per_sweep']:.2f} ms  " + "  ".join(
            f"N={n}: {sp[n]['ms_max_over_ranks']:.2f} ms ({sp[n]['implied_speedup']:.2f}x)" for n in ("2", "4", "8") if n in sp))
