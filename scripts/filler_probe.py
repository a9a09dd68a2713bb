"""Diagnostic: rank R's shard of 8 (all four families) as in bench.time_replay
(stitch-heavy families first on higher-priority streams), vs the same plus each
family's last FRAC of scenarios split off at MULT x the segments and launched
after all bulk parts, at priority MODE (same = its family's, hi = highest,
lo = lowest)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402


def split(tr, S0):
    a0 = int(tr.offsets[S0])
    bulk = orj.Trace(tr.offsets[:S0 + 1].clone(), tr.arrival[:a0], tr.dist[:a0], tr.true_bin[:a0], tr.slo[:S0],
                     tr.bucket[:S0], tr.num_buckets)
    tail = orj.Trace(tr.offsets[S0:] - a0, tr.arrival[a0:], tr.dist[a0:], tr.true_bin[a0:], tr.slo[S0:],
                     tr.bucket[S0:], tr.num_buckets)
    return bulk, tail


def run(fams, parts, prios, reps=5):
    main_s = torch.cuda.current_stream()
    wss = [torch.empty(max(orj.replay_seg_workspace_bytes(tr, g), 1), dtype=torch.uint8, device="cuda")
           for _, tr, g in parts]
    streams = [torch.cuda.Stream(priority=p) for p in prios]
    ts = []
    for rep in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main_s)
        for (i, tr, g), s, ws in zip(parts, streams, wss):
            s.wait_event(e0)
            orj.replay_trace(fams[i].store, fams[i].profile, tr, stream=s, segments=g, workspace=ws)
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            main_s.wait_event(ev)
        e1.record(main_s)
        torch.cuda.synchronize()
        if rep:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    sys.argv = [sys.argv[0]]
    args = bench.parse()
    r = int(os.environ.get("RANK_", "6"))
    G = 24
    fams = bench.build_replay(args, r, 8, torch.device("cuda", 0))
    names = [f.tf.fam.name for f in fams]
    order = [names.index(n) for n in ("rdi", "gpt", "skipnet", "static")]
    lo, hi = torch.cuda.Stream.priority_range()
    pr_of = {i: min(lo, hi + order.index(i)) for i in range(4)}
    base = run(fams, [(i, fams[i].trace, G) for i in order], [pr_of[i] for i in order])
    print(f"rank {r} base G={G}: {base:.3f} ms", flush=True)
    for frac in (0.125, 0.25):
        for mult in (2, 4):
            for mode in ("same", "hi"):
                parts, prios = [], []
                tails = []
                for i in order:
                    S = fams[i].trace.num_scenarios
                    nt = int(round(S * frac))
                    b_, t_ = split(fams[i].trace, S - nt)
                    parts.append((i, b_, G))
                    prios.append(pr_of[i])
                    tails.append((i, t_, G * mult))
                for (i, t_, g) in tails:
                    parts.append((i, t_, g))
                    prios.append(pr_of[i] if mode == "same" else hi)
                print(f"  frac {frac} mult {mult} {mode}: {run(fams, parts, prios):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
