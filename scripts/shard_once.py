"""Profiling target: rank RANK_'s round-robin shard of WORLD (the bench's C5
families), each family's segmented replay once after a warm-up, one after the
other on the default stream (for ncu launch lists).  Env: WORLD (8), RANK_ (0),
SEGS (bench --replay-segments spec, default auto)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402


def main():
    sys.argv = [sys.argv[0]]
    args = bench.parse()
    dev = torch.device("cuda", 0)
    world, r = int(os.environ.get("WORLD", "8")), int(os.environ.get("RANK_", "0"))
    spec = os.environ.get("SEGS", "auto")
    fams = bench.build_replay(args, r, world, dev)
    for f in fams:
        g = bench.replay_segments(bench.family_segments(spec, f.tf.fam.name), f.trace.num_scenarios,
                                  f.trace.num_arrivals // max(f.trace.num_scenarios, 1))
        ws = torch.empty(max(orj.replay_seg_workspace_bytes(f.trace, g), 1), dtype=torch.uint8, device=dev)
        for _ in range(2):
            orj.replay_trace(f.store, f.profile, f.trace, segments=g, workspace=ws)
        torch.cuda.synchronize()
        print(f.tf.fam.name, "segments", g, orj.replay_seg_stats(ws), flush=True)


if __name__ == "__main__":
    main()
