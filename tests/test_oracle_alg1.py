"""Pins of oracle/alg1.py (Alg. 1 replay): hand-traced
cases, exact thresholds, and invariants.  The hand traces are derived in the
comments from the paper's definitions (not from any implementation)."""
import math

import numpy as np

import gen
from oracle import alg1
from oracle import priority as pr
from paper_2209_00159_b200 import policy


def _one_app_point_mass():
    # one application, every request in bin 1, B = 4; kmax = 3 (the window holds 3)
    counts = np.array([[8, 0, 0, 0]])
    a = np.array([0, 0, 0], np.int64)
    w = np.array([10, 15, 22], np.int64)
    return counts, a, w


def test_thresholds_hand_values():
    counts, a, w = _one_app_point_mass()
    # L_bs uniform on (0, w_bs]: E = 5, 7.5, 11 -> ceil 5, 8, 11
    assert list(alg1.size_thresholds(counts, a, w)) == [5, 8, 11]


def test_two_identical_requests_pop_as_one_batch():
    """SPEC scheduler example: 2 identical requests, S = {1, 2}, both feasible
    for bs = 2 -> one batch of 2.  Q_1 = Q_2 = {r1, r2}, D_Q1 = D_Q2 -> the tie
    goes to the larger bs (bs 3 needs 3 members); duration a_2 + w_2 * 1 = 15 <= 100:
    both finish."""
    counts, a, w = _one_app_point_mass()
    thr = alg1.size_thresholds(counts, a, w)
    out = alg1.replay(counts, a, w, 0.01, np.array([0, 2]), np.array([0, 0]), np.zeros(2, np.int32),
                      np.ones(2, np.int16), np.array([100]), thr, want_log=True)
    assert list(out["counters"][0]) == [2, 2, 0, 0, 1, 15, 15]
    assert list(out["log"][:2]) == [0b11, 0]


def test_idle_worker_then_pair():
    """r1 arrives at -94, r2 and r3 at 0; SLO 100; every true bin 1.
    t = -94: window {r1} -> bs 1 (one member), duration 10, ends -84 <= 6: finished.
    t = 0 (idle jump): {r2, r3}, slack 100 >= thr_2 = 8: Q_1 = Q_2, D_Q1 = D_Q2 -> the
    tie goes to bs 2; duration 15, ends 15 <= 100: both finish.
    Counters: total 3, finished 3, dropped 0, late 0, batches 2, busy 25, span 15 + 94."""
    counts, a, w = _one_app_point_mass()
    thr = alg1.size_thresholds(counts, a, w)
    out = alg1.replay(counts, a, w, 0.01, np.array([0, 3]), np.array([-94, 0, 0]), np.zeros(3, np.int32),
                      np.ones(3, np.int16), np.array([100]), thr, want_log=True)
    assert list(out["counters"][0]) == [3, 3, 0, 0, 2, 25, 109]
    assert list(out["log"][:3]) == [0b1, 0b11, 0]


def test_popbatch_by_priority_skips_the_earliest_deadline():
    """SLO 49; r0 at 0 with true bin 4 runs alone over (0, 40] (r1..r3 arrive later).
    r1, r2, r3 arrive at 1, 6, 31: at t = 40 their slacks are 10, 15, 40 (all >= thr_1 = 5
    and >= thr_2 = 8), so Q_1 = Q_2 = {r1, r2, r3}; Q_3 = {r2, r3} (10 < thr_3 = 11) is
    too small for bs 3; D_Q1 = D_Q2 -> bs = 2.
    Eq. 2 with L_2 ~ U(0, 15], b = 0.01 (common factor h / (b E[L]) dropped):
      r1: sigma 10 < 15, partial bin: 1 - e^{-0.10}              = 0.0952
      r2: sigma 15 = l2, full bin:    (e^{0.15} - 1) e^{-0.15}   = 0.1393
      r3: sigma 40, full bin:         (e^{0.15} - 1) e^{-0.40}   = 0.1085
    PopBatch pops r2 and r3 (mask 0b110), not the earliest deadline; duration
    15 -> t = 55: r2 (D = 55, inclusive) and r3 (D = 80) finish.  r1 stays
    pending: at t = 55 its slack is -5 < thr_1 -> dropped.
    Counters: total 4, finished 3, dropped 1, late 0, batches 2, busy 55, span 55."""
    counts, a, w = _one_app_point_mass()
    thr = alg1.size_thresholds(counts, a, w)
    arr = np.array([0, 1, 6, 31])
    tb = np.array([4, 1, 1, 1], np.int16)
    out = alg1.replay(counts, a, w, 0.01, np.array([0, 4]), arr, np.zeros(4, np.int32), tb, np.array([49]), thr,
                      want_log=True)
    assert list(out["counters"][0]) == [4, 3, 1, 0, 2, 55, 55]
    assert list(out["log"][:3]) == [0b1, 0b110, 0]


def test_deadline_tie_goes_to_the_largest_feasible_size():
    """SLO 100; r0 at -100 with true bin 4 runs over (-100, -60]; r1 at -94, r2 and
    r3 at -70.  t = -60: slacks 66, 90, 90 >= thr_3 = 11, so Q_1 = Q_2 = Q_3 = all
    three and D_Q1 = D_Q2 = D_Q3 -> the tie goes to bs 3: one batch of all three,
    duration 22 -> t = -38.  All finish.
    Counters: total 4, finished 4, dropped 0, late 0, batches 2, busy 62, span 62."""
    counts, a, w = _one_app_point_mass()
    thr = alg1.size_thresholds(counts, a, w)
    out = alg1.replay(counts, a, w, 0.01, np.array([0, 4]), np.array([-100, -94, -70, -70]), np.zeros(4, np.int32),
                      np.array([4, 1, 1, 1], np.int16), np.array([100]), thr, want_log=True)
    assert list(out["counters"][0]) == [4, 4, 0, 0, 2, 62, 62]
    assert list(out["log"][:3]) == [0b1, 0b111, 0]


def test_thresholds_exact_vs_float_and_host_policy():
    fam = gen.skipnet_family(gen.SEED_BASE + 930)
    prof = gen.eq3_half(fam, 32)
    wts = np.linspace(0.5, 2.0, fam.D).astype(np.float32)
    thr = alg1.size_thresholds(fam.counts, prof.a, prof.w, wts)
    # float evaluation of the same E[L_bs] (exact counts): ceil agrees unless within 1e-6 of an integer
    for k in range(32):
        e = pr.expected_latency(pr.batch_latency_pmf(fam.counts, k + 1, wts), prof.a[k], prof.w[k])
        if abs(e - round(e)) > 1e-6:
            assert thr[k] == math.ceil(e)
    assert (np.diff(thr) >= 0).all()
    # the product's host-side policy builder computes the same integers
    assert np.array_equal(policy.alg1_size_thresholds(fam.counts, prof.a, prof.w, wts), thr)


def test_replay_invariants_and_follow_own_log():
    tf = gen.c5_trace_family("gpt")
    gids = np.arange(3, dtype=np.uint64)
    n = 600
    arr, dist, tb = gen.trace_host(tf, gids, n)
    off = np.arange(4, dtype=np.int64) * n
    slo = np.array([tf.slo_of_bucket(b) for b in (0, 3, 7)], np.int64)
    thr = alg1.size_thresholds(tf.fam.counts, tf.profile.a, tf.profile.w)
    b = 1.0 / tf.fam.mean_ticks()
    free = alg1.replay(tf.fam.counts, tf.profile.a, tf.profile.w, b, off, arr, dist, tb, slo, thr, want_log=True)
    c = free["counters"]
    assert (c[:, 0] == c[:, 1] + c[:, 2] + c[:, 3]).all()
    assert (c[:, 5] <= c[:, 6]).all()
    fol = alg1.replay(tf.fam.counts, tf.profile.a, tf.profile.w, b, off, arr, dist, tb, slo, thr,
                      follow_log=free["log"])
    assert (fol["ties"][:, 2] == -1).all() and (fol["ties"][:, 1] == 0).all()
    assert np.array_equal(fol["counters"], c)
    # a wrong mask (pop the last member instead of the first of a 2-pop) is flagged
    bad = free["log"].copy()
    idx = np.nonzero(bad == 0b11)[0]
    if len(idx):
        bad[idx[0]] = 0b101
        assert alg1.replay(tf.fam.counts, tf.profile.a, tf.profile.w, b, off, arr, dist, tb, slo, thr,
                           follow_log=bad)["ties"][:, 2].max() >= 0


def test_abi_thresholds_equal_exact_rationals():
    """orloj_alg1_size_thresholds (C ABI, big-integer arithmetic) equals the
    oracle's exact-rational evaluation on random histograms with empty bins,
    unequal totals, zero and non-dyadic weights, point masses, kmax 32; and
    orloj_expected_latency_thresholds equals ceil of the exact rational
    a_1 + w_1 sum_i i c_i / sum_i c_i."""
    from fractions import Fraction
    rng = np.random.default_rng(gen.SEED_BASE + 931)
    for trial in range(12):
        D = int(rng.integers(1, 9))
        B = int(rng.choice([4, 8, 16, 64]))
        counts = rng.integers(0, 1 << int(rng.integers(3, 31)), size=(D, B)).astype(np.uint32)
        counts[rng.random((D, B)) < 0.4] = 0
        counts[:, int(rng.integers(0, B))] += 1
        if trial % 4 == 0:
            counts[0] = 0
            counts[0, B // 2] = 5                        # a point mass
        a = np.cumsum(rng.integers(0, 3000, 32)).astype(np.int64)
        w = np.cumsum(rng.integers(0, 500, 32)).astype(np.int64) + 1
        wts = None if trial % 3 == 0 else rng.random(D) * 3
        if wts is not None and D > 1:
            wts[0] = 0.0
        ref = alg1.size_thresholds(counts, a, w, wts)
        got = policy.alg1_size_thresholds(counts, a, w, wts)
        assert np.array_equal(got, ref), trial
        el = policy.expected_latency_thresholds(counts, a, w)
        for d in range(D):
            e = Fraction(int(a[0])) + Fraction(int(w[0]) * sum((i + 1) * int(c) for i, c in enumerate(counts[d])),
                                                int(counts[d].sum()))
            assert el[d] == math.ceil(e)


def test_abi_thresholds_errors():
    import pytest
    from paper_2209_00159_b200 import OrlojError
    counts = np.ones((2, 8), np.uint32)
    counts[1] = 0
    with pytest.raises(OrlojError, match="COLD_START"):
        policy.alg1_size_thresholds(counts, [0], [1])
    with pytest.raises(OrlojError, match="COLD_START"):
        policy.expected_latency_thresholds(counts, [0], [1])
    with pytest.raises(OrlojError, match="INVALID"):
        policy.alg1_size_thresholds(np.ones((2, 8)), [0], [1], weights=[0.0, 0.0])
