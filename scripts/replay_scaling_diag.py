"""Replay strong-scaling diagnosis (one GPU): time each C5 family alone for the
rank-0 shard of N GPUs, a single scenario alone (the decision-chain latency
floor), and the decisions per scenario, to see what sets the 8-GPU time."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402
from paper_2209_00159_b200 import parallel  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
nb = len(gen.BUCKET_SLO_MULTS)
world = int(os.environ.get("DIAG_WORLD", "8"))
u = np.arange(nb * gen.C5_SEEDS_PER_BUCKET)
mine = parallel.shard_round_robin(u // nb, 0, world)
for name in gen.C5_FAMILIES:
    f = wl.C5Family(name, local_ids=mine)
    ms = timed(lambda: orj.replay_trace(f.store, f.profile, f.trace))
    pb, log = orj.replay_trace(f.store, f.profile, f.trace, decision_log=True)
    torch.cuda.synchronize()
    # decisions per scenario from the log (0-terminated per scenario)
    lg = log.cpu().numpy()
    S, n = f.num_scenarios, f.n_arr
    dec = np.array([int(np.argmax(lg[s * (n + 1):(s + 1) * (n + 1)] == 0)) for s in range(S)])
    worst = int(np.argmax(dec))
    one = wl.C5Family(name, local_ids=mine[[worst]])
    ms1 = timed(lambda: orj.replay_trace(one.store, one.profile, one.trace))
    out[name] = {"scenarios": S, "ms_shard": ms, "decisions_mean": float(dec.mean()), "decisions_max": int(dec.max()),
                 "worst_bucket": int(f.bucket_np[worst]), "ms_worst_alone": ms1,
                 "ns_per_decision_alone": 1e6 * ms1 / dec.max()}
    print(name, json.dumps(out[name]), flush=True)
print(json.dumps(out))
