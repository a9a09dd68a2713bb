"""Diagnostic: the 8-way shard proxy (bench.shard_proxy's per-rank sweep) for a
few ranks at several segment specs (bench.family_segments syntax), median of 3."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    args = bench.parse.__wrapped__() if hasattr(bench.parse, "__wrapped__") else None
    sys.argv = [sys.argv[0]]
    args = bench.parse()
    dev = torch.device("cuda", 0)
    specs = os.environ.get("SPECS", "auto;rdi=16,auto;rdi=12,auto;rdi=32,auto").split(";")
    ranks = [int(x) for x in os.environ.get("RANKS", "0,6").split(",")]
    for r in ranks:
        sf = bench.build_replay(args, r, 8, dev)
        for spec in specs:
            ts = []
            for _ in range(3):
                ms, _, _ = bench.time_replay(sf, 1, dev, lambda: None, lambda x: x, reduce=False, segments=spec)
                ts.append(ms)
            print(f"rank {r} spec {spec}: {np.median(ts):.3f} ms  segs {bench.time_replay.segments} "
                  f"order {bench.time_replay.launch_order} "
                  f"stitch {[s['stitch_decisions'] if s else 0 for s in bench.time_replay.stats]}", flush=True)
        del sf


if __name__ == "__main__":
    main()
