"""Small end-to-end exercise of every kernel, run under compute-sanitizer by
tests/test_gpu_sanitizer.py (memcheck, racecheck, synccheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402


def main():
    # C1 pick + score (shared-memory store path)
    c = gen.config1()
    st = orj.HistogramStore.from_counts(c.fam.counts, c.fam.bin_ticks)
    pr = orj.LatencyProfile(c.profile.a, c.profile.w)
    q = wl.device_queues(c.queues)
    q.validate(st)
    orj.pick_batch(st, pr, q)
    orj.score_batches(st, pr, q, want_P=True, want_EL=True)
    # small C3-shaped queues (TMA ring path, 256 bins, kmax 64)
    c3 = gen.config3(Q=16, n=80, kmax=64, T=64)
    st3 = wl.c3_store(c3)
    st3.validate()
    q3 = wl.device_queues(c3.queues)
    orj.pick_batch(st3, wl.profile(c3.profile), q3)
    orj.score_batches(st3, wl.profile(c3.profile), q3, want_P=True, want_EL=True)
    # replay (8 scenarios x 500 arrivals)
    f = wl.C5Family("skipnet", local_ids=np.arange(8), n_arr=500)
    f.trace.validate(f.store)
    orj.replay_trace(f.store, f.profile, f.trace, decision_log=True)
    torch.cuda.synchronize()
    print("sanitize case OK")


if __name__ == "__main__":
    main()
