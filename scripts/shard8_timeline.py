"""Diagnostic: completion time of each family in one concurrent sweep of rank
R's shard of 8 (events on each family's stream; both replay passes inside), and
each family's time when run alone."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402


def main():
    sys.argv = [sys.argv[0]]
    args = bench.parse()
    dev = torch.device("cuda", 0)
    r = int(os.environ.get("RANK_", "6"))
    G = int(os.environ.get("SEGS", "24"))
    fams = bench.build_replay(args, r, 8, dev)
    wss = [torch.empty(max(orj.replay_seg_workspace_bytes(f.trace, G), 1), dtype=torch.uint8, device=dev) for f in fams]
    names = [f.tf.fam.name for f in fams]
    lo, hi = torch.cuda.Stream.priority_range()
    order = [names.index(n) for n in os.environ.get("ORDER", "rdi,gpt,skipnet,static").split(",")]
    mode = os.environ.get("PRIO", "ranked")  # ranked | flat | rdi
    pr = {"ranked": lambda i: min(lo, hi + order.index(i)), "flat": lambda i: lo,
          "rdi": lambda i: hi if names[i] == "rdi" else lo}[mode]
    streams = [torch.cuda.Stream(dev, priority=pr(i)) for i in range(len(fams))]
    main_s = torch.cuda.current_stream()
    for rep in range(4):
        start = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in fams]
        start.record(main_s)
        for i in order:
            streams[i].wait_event(start)
            orj.replay_trace(fams[i].store, fams[i].profile, fams[i].trace, stream=streams[i], segments=G,
                             workspace=wss[i])
            ends[i].record(streams[i])
        torch.cuda.synchronize()
        if rep:
            print("concurrent", mode, G, ":", {names[i]: round(start.elapsed_time(ends[i]), 3) for i in range(len(fams))}, flush=True)
    for i in range(len(fams)):
        ts = []
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main_s)
            orj.replay_trace(fams[i].store, fams[i].profile, fams[i].trace, segments=G, workspace=wss[i])
            e1.record(main_s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print("alone", names[i], round(float(np.median(ts)), 3), flush=True)


if __name__ == "__main__":
    main()
