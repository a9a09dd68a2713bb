"""Window-size statistics of the C5 sweep (diagnostic): run with
ORLOJ_LIB=build_variants/liborloj_stats.so (built with -DORLOJ_REPLAY_STATS)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402

out = {}
for name in gen.C5_FAMILIES:
    f = wl.C5Family(name)
    ws = torch.zeros(orj.replay_seg_workspace_bytes(f.trace, 8), dtype=torch.uint8, device="cuda")
    tab, _ = orj.replay_trace(f.store, f.profile, f.trace, segments=8, workspace=ws)
    torch.cuda.synchronize()
    v = ws[:256].view(torch.int64).cpu().numpy()
    dec = int(tab[:, 4].sum())
    out[name] = {"decisions": dec, "maxplus": int(v[5]), "carried_scans": int(v[6]),
                 "wc_hist": [int(x) for x in v[7:32]]}
    print(json.dumps({name: out[name]}), flush=True)
    del f
