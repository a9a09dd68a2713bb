"""Diagnostic: is one launch over all scenarios faster than four concurrent
launches of a quarter each?  SkipNet, 1,024 scenarios (the size of a rank's
shard of 8 over all four families), G segments: one replay_trace call, vs the
same scenarios split into four calls on four streams."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[1:]))


def main():
    G = int(os.environ.get("SEGS", "24"))
    fam = os.environ.get("FAM", "skipnet")
    nb = len(gen.BUCKET_SLO_MULTS)
    allf = wl.C5Family(fam, local_ids=np.arange(nb * 128))    # 1,024 scenarios
    parts = [wl.C5Family(fam, local_ids=np.arange(nb * 128)[i::4]) for i in range(4)]
    ws = torch.empty(max(orj.replay_seg_workspace_bytes(allf.trace, G), 1), dtype=torch.uint8, device="cuda")
    wss = [torch.empty(max(orj.replay_seg_workspace_bytes(f.trace, G), 1), dtype=torch.uint8, device="cuda") for f in parts]
    streams = [torch.cuda.Stream() for _ in parts]
    one = timed(lambda: orj.replay_trace(allf.store, allf.profile, allf.trace, segments=G, workspace=ws))
    main_s = torch.cuda.current_stream()

    def four():
        ev = torch.cuda.Event()
        ev.record(main_s)
        for f, s, w in zip(parts, streams, wss):
            s.wait_event(ev)
            orj.replay_trace(f.store, f.profile, f.trace, segments=G, workspace=w, stream=s)
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            main_s.wait_event(e)
    four_ms = timed(four)
    print(f"{fam} G={G}: one launch {one:.3f} ms, four concurrent quarters {four_ms:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
