"""Replay one C5 family's rank-0 shard of DIAG_WORLD GPUs twice (profiling target); DIAG_SEGMENTS
segments per scenario (1 = plain kernel)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402
from paper_2209_00159_b200 import parallel  # noqa: E402

nb = len(gen.BUCKET_SLO_MULTS)
world = int(os.environ.get("DIAG_WORLD", "8"))
u = np.arange(nb * gen.C5_SEEDS_PER_BUCKET)
mine = parallel.shard_round_robin(u // nb, 0, world)
f = wl.C5Family(os.environ.get("DIAG_FAMILY", "skipnet"), local_ids=mine,
                n_arr=int(os.environ.get("DIAG_ARRIVALS", "20000")))
G = int(os.environ.get("DIAG_SEGMENTS", "1"))
ws = torch.empty(max(orj.replay_seg_workspace_bytes(f.trace, G), 1), dtype=torch.uint8, device="cuda")
for _ in range(2):
    orj.replay_trace(f.store, f.profile, f.trace, segments=G, workspace=ws)
torch.cuda.synchronize()
print("done")
