"""Diagnostic: a rank's 1,024-scenario SkipNet shard as one launch at G
segments, vs a bulk part at G on a high-priority stream plus the last scenarios
at finer segments on a low-priority stream (the filler drains the tail)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402
from merge_probe import timed  # noqa: E402


def main():
    fam = os.environ.get("FAM", "skipnet")
    nb = len(gen.BUCKET_SLO_MULTS)
    ids = np.arange(nb * 128)
    G = 24
    allf = wl.C5Family(fam, local_ids=ids)
    ws = torch.empty(max(orj.replay_seg_workspace_bytes(allf.trace, G), 1), dtype=torch.uint8, device="cuda")
    one = timed(lambda: orj.replay_trace(allf.store, allf.profile, allf.trace, segments=G, workspace=ws))
    print(f"{fam}: one launch G={G}: {one:.3f} ms", flush=True)
    lo, hi = torch.cuda.Stream.priority_range()
    for frac, gt in ((0.125, 48), (0.125, 96), (0.25, 48), (0.25, 96), (0.0625, 128)):
        nt = int(len(ids) * frac)
        # the tail takes scenarios from every bucket (strided) so both parts keep the mix
        tail_ids = ids[::int(1 / frac)][:nt]
        bulk_ids = np.setdiff1d(ids, tail_ids)
        fb, ft = wl.C5Family(fam, local_ids=bulk_ids), wl.C5Family(fam, local_ids=tail_ids)
        wb = torch.empty(max(orj.replay_seg_workspace_bytes(fb.trace, G), 1), dtype=torch.uint8, device="cuda")
        wt = torch.empty(max(orj.replay_seg_workspace_bytes(ft.trace, gt), 1), dtype=torch.uint8, device="cuda")
        sb, st = torch.cuda.Stream(priority=hi), torch.cuda.Stream(priority=lo)
        main_s = torch.cuda.current_stream()

        def two():
            ev = torch.cuda.Event()
            ev.record(main_s)
            sb.wait_event(ev)
            st.wait_event(ev)
            orj.replay_trace(fb.store, fb.profile, fb.trace, segments=G, workspace=wb, stream=sb)
            orj.replay_trace(ft.store, ft.profile, ft.trace, segments=gt, workspace=wt, stream=st)
            for s in (sb, st):
                e = torch.cuda.Event()
                e.record(s)
                main_s.wait_event(e)
        print(f"  bulk G={G} + tail {frac:.3f} at G={gt} (low priority): {timed(two):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
