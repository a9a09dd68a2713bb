"""Diagnostic (variant library built with ORLOJ_REPLAY_TIMELINE, loaded via
ORLOJ_LIB): one concurrent sweep of rank R's shard of N (the bench's launch:
4 families on 4 streams, stitch-heavy first) and, per family, the %globaltimer
spans of every first-pass item and every stitch, plus the number of items in
flight over time.  Env: WORLD (8), RANK_ (0), SEGS (auto)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402

SEG_BYTES = 3136      # sizeof(ReplaySeg) with the timeline fields
TL_OFF = 3088         # offset of tl[4]


def main():
    sys.argv = [sys.argv[0]]
    args = bench.parse()
    dev = torch.device("cuda", 0)
    world, r = int(os.environ.get("WORLD", "8")), int(os.environ.get("RANK_", "0"))
    fams = bench.build_replay(args, r, world, dev)
    names = [f.tf.fam.name for f in fams]
    spec = os.environ.get("SEGS", "auto,last=auto")
    segs = [bench.replay_segments(bench.family_segments(spec, f.tf.fam.name), f.trace.num_scenarios,
                                  f.trace.num_arrivals // max(f.trace.num_scenarios, 1)) for f in fams]
    wss = [torch.empty(orj.replay_seg_workspace_bytes(f.trace, g), dtype=torch.uint8, device=dev)
           for f, g in zip(fams, segs)]
    lo, hi = torch.cuda.Stream.priority_range()
    main_s = torch.cuda.current_stream()
    order = list(range(len(fams)))
    streams = [torch.cuda.Stream(dev) for _ in fams]
    out = {}
    for rep in range(3):
        start = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in fams]
        start.record(main_s)
        for i in order:
            streams[i].wait_event(start)
            orj.replay_trace(fams[i].store, fams[i].profile, fams[i].trace, stream=streams[i], segments=segs[i],
                             workspace=wss[i])
            ends[i].record(streams[i])
        torch.cuda.synchronize()
        if rep == 0:
            work = [orj.replay_seg_stats(ws)["stitch_decisions"] for ws in wss]
            order = sorted(range(len(fams)), key=lambda i: -work[i])
            rank_of = {i: k for k, i in enumerate(order)}
            streams = [torch.cuda.Stream(dev, priority=min(lo, hi + rank_of[i])) for i in range(len(fams))]
            i = order[-1]
            segs[i] = bench.last_segments(spec, segs[i], fams[i].trace.num_scenarios)  # as the bench
            wss[i] = torch.empty(orj.replay_seg_workspace_bytes(fams[i].trace, segs[i]), dtype=torch.uint8,
                                 device=dev)
            continue
        out[f"rep{rep}_ms_end"] = {names[i]: round(start.elapsed_time(ends[i]), 3) for i in range(len(fams))}
    spans = {}
    t0 = None
    for i, (f, ws) in enumerate(zip(fams, wss)):
        S, G = f.trace.num_scenarios, segs[i]
        raw = ws[256:256 + S * G * SEG_BYTES].cpu().numpy().reshape(S * G, SEG_BYTES)
        tl = raw[:, TL_OFF:TL_OFF + 32].copy().view(np.int64).reshape(S * G, 4)
        sm = raw[:, TL_OFF + 32:TL_OFF + 40].copy().view(np.int32).reshape(S * G, 2)
        p1 = tl[:, :2]
        p2 = tl.reshape(S, G, 4)[:, 0, 2:]
        spans[names[i]] = (p1, p2, sm[:, 0])
        m = p1[:, 0].min()
        t0 = m if t0 is None else min(t0, m)
    res = {"world": world, "rank": r, "segments": segs, "order": [names[i] for i in order], **out}
    for name, (p1, p2, sm) in spans.items():
        d1 = (p1[:, 1] - p1[:, 0]) / 1e6
        res[name] = {"items": int(len(p1)),
                     "p1_start_ms": [round(float(x), 3) for x in np.percentile((p1[:, 0] - t0) / 1e6, [0, 50, 90, 100])],
                     "p1_end_ms": [round(float(x), 3) for x in np.percentile((p1[:, 1] - t0) / 1e6, [0, 50, 90, 100])],
                     "p1_item_ms": [round(float(x), 3) for x in np.percentile(d1, [0, 10, 50, 90, 99, 100])],
                     "p2_start_ms": [round(float(x), 3) for x in np.percentile((p2[:, 0] - t0) / 1e6, [0, 50, 100])],
                     "p2_end_ms": [round(float(x), 3) for x in np.percentile((p2[:, 1] - t0) / 1e6, [0, 50, 90, 100])],
                     "p2_item_ms": [round(float(x), 3) for x in np.percentile((p2[:, 1] - p2[:, 0]) / 1e6, [0, 50, 90, 100])]}
        # item duration vs segment index (segment-major cost profile)
        G = len(p1) // len(p2)
        res[name]["p1_ms_by_segment"] = [round(float(x), 3) for x in d1.reshape(-1, G).mean(axis=0)]
    # items in flight over time (0.25 ms bins), both passes, all families
    tmax = max(int(max(p1[:, 1].max(), p2[:, 1].max()) - t0) for p1, p2, _ in spans.values())
    edges = np.arange(0, tmax + 250_000, 250_000)
    fl1 = np.zeros(len(edges), np.int64)
    fl2 = np.zeros(len(edges), np.int64)
    for p1, p2, _ in spans.values():
        for arr, fl in ((p1, fl1), (p2, fl2)):
            a = np.searchsorted(edges, arr[:, 0] - t0)
            b = np.searchsorted(edges, arr[:, 1] - t0)
            np.add.at(fl, a, 1)
            np.add.at(fl, b, -1)
    res["inflight_p1_per_0.25ms"] = np.cumsum(fl1).tolist()
    res["inflight_p2_per_0.25ms"] = np.cumsum(fl2).tolist()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
