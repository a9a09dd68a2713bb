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
    orj.replay_trace(f.store, f.profile, f.trace, objective="finish_rate")
    # segmented replay (speculative segments + stitch), with and without the log
    orj.replay_trace(f.store, f.profile, f.trace, decision_log=True, segments=5)
    orj.replay_trace(f.store, f.profile, f.trace, segments=3, objective="finish_rate")
    orj.replay_trace(f.store, f.profile, f.trace, decision_log=True, segments=200)  # segments of 2-3 arrivals
    # Alg. 1 policy (priority tables inside the replay kernel)
    from paper_2209_00159_b200 import policy
    pt = orj.PriorityTable(f.store, f.profile, f.profile.kmax, 1.0 / f.tf.fam.mean_ticks())
    thr = torch.from_numpy(policy.alg1_size_thresholds(f.tf.fam.counts, f.tf.profile.a, f.tf.profile.w)).cuda()
    orj.replay_trace(f.store, f.profile, f.trace, decision_log=True, objective="alg1", priority=pt,
                     size_thresholds=thr)
    # priorities (+ steps), PopBatch, model variants, profiler on the C1 queue
    tab = orj.PriorityTable(st, pr, 4, 1e-3)
    lp = tab.scores(q)
    tab.scores(q, steps=([0, 500], [1.0, 2.0]))
    tab.pop(q, lp, torch.tensor([3], dtype=torch.int32, device="cuda"))
    for interp in (False, True):
        orj.ScoreModel.eq3(pr, st.num_bins, interpolate=interp, steps=([0, 300], [1.0, 1.5])).score(st, q)
    # round-2 paths: short-queue full-queue build (C4 shape), priority TIER 0 / 1 with the
    # vector member map and both PopBatch paths, the model edge kernel (grid rows, a
    # non-grid row, several steps)
    c4 = gen.config4(Q=40)
    st4 = orj.HistogramStore.from_counts(c4.fam.counts, c4.fam.bin_ticks)
    orj.pick_batch(st4, wl.profile(c4.profile), wl.device_queues(c4.queues))
    cp = gen.config_priority(Q=12, n=256)
    cp.queues.offsets[6:] -= 3  # a short queue and unaligned chunks next to full ones
    stp = orj.HistogramStore.from_counts(cp.fam.counts, cp.fam.bin_ticks)
    qp = wl.device_queues(cp.queues)
    for b in (1.0 / cp.fam.mean_ticks(), 50.0 / cp.fam.mean_ticks()):
        tp = orj.PriorityTable(stp, wl.profile(cp.profile), 32, b)
        lpp = tp.scores(qp)
        tp.pop(qp, lpp, torch.full((cp.queues.Q,), 32, dtype=torch.int32, device="cuda"))
        tp.pop(qp, torch.zeros_like(lpp), torch.full((cp.queues.Q,), 5, dtype=torch.int32, device="cuda"))
    c2 = gen.config2(Q=16)
    st2 = orj.HistogramStore.from_counts(c2.fam.counts, c2.fam.bin_ticks)
    q2 = wl.device_queues(c2.queues)
    m = np.arange(c2.fam.B + 1, dtype=np.int64)
    eq3 = c2.profile.a[:, None] + c2.profile.w[:, None] * m[None, :]
    logm = eq3.copy()
    logm[3] = c2.profile.a[3] + c2.profile.w[3] * np.round(c2.fam.B * (2.0 ** (4.0 * m / c2.fam.B) - 1.0) / 15.0).astype(np.int64)
    for tab_, st_ in ((eq3, None), (eq3, ([0, 300], [1.0, 1.5])), (logm, None), (logm, ([0, 300], [1.0, 1.5]))):
        orj.ScoreModel(tab_, steps=st_).score(st2, q2)
    prof = orj.Profiler(st.num_dists, st.num_bins, st.bin_ticks)
    prof.add(torch.tensor([0, 1, 2], dtype=torch.int32, device="cuda"),
             torch.tensor([5, 1500, 99999], dtype=torch.int64, device="cuda"))
    torch.cuda.synchronize()
    print("sanitize case OK")


if __name__ == "__main__":
    main()
