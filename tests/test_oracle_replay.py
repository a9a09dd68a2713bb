"""Oracle pins for the trace replay (readings A9, A11, A15-A17).

* hand cases: tests/test_oracle_examples.py.
* invariants: conservation finished + dropped + late = total;
  non-preemption busy <= span; determinism; decision log
  well formed; follow mode with the oracle's own log reproduces it.
* point masses: the replay must equal a textbook constant-latency planner
  replay that knows every member's time exactly and counts on-time members
  with integers only (no probabilities).
"""
import numpy as np
import pytest

import gen
import oracle


def _small_trace(tf, S=6, n=400, gid0=0):
    gids = np.arange(gid0, gid0 + S, dtype=np.uint64)
    arr, dist, tb = gen.trace_host(tf, gids, n)
    off = np.arange(S + 1, dtype=np.int64) * n
    slo = np.array([tf.slo_of_bucket(b % 8) for b in range(S)], np.int64)
    return off, arr, dist, tb, slo


@pytest.mark.parametrize("fam", gen.C5_FAMILIES)
def test_replay_invariants(fam):
    tf = gen.c5_trace_family(fam)
    off, arr, dist, tb, slo = _small_trace(tf)
    F = oracle.cdf(tf.fam.counts)
    r = oracle.replay(F, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo, want_log=True)
    c = r["counters"]
    assert (c[:, 0] == np.diff(off)).all()
    assert (c[:, 1] + c[:, 2] + c[:, 3] == c[:, 0]).all()
    assert (c[:, 5] <= c[:, 6]).all()
    assert (c[:, 4] >= 1).all()
    log = r["log"]
    for s in range(len(slo)):
        base = off[s] + s
        seg = log[base: base + c[s, 4] + 1]
        assert seg[-1] == 0 and (seg[:-1] >= 1).all() and (seg[:-1] <= tf.profile.kmax).all()
    # determinism
    r2 = oracle.replay(F, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo, want_log=True)
    assert (r2["counters"] == c).all() and (r2["log"] == log).all()
    # follow mode with its own log is a no-op
    r3 = oracle.replay(F, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo, follow_log=log)
    assert (r3["counters"] == c).all()
    assert (r3["ties"][:, 1] == 0).all() and (r3["ties"][:, 2] == -1).all()


def _planner_replay(bins_of_dist, a, w, kmax, arrival, dist, tb, slo):
    """Textbook replay with exactly known times (point masses): pick the k that
    maximises the integer count of on-time members (smallest on ties)."""
    n = len(arrival)
    t = None
    cursor, carry = 0, []
    fin = drop = late = bat = busy = 0
    while cursor < n or carry:
        if not carry and (t is None or arrival[cursor] > t):
            t = int(arrival[cursor])
        live = list(carry)
        win = []
        for r in live:
            if t + a[0] + w[0] * bins_of_dist[dist[r]] > arrival[r] + slo:
                drop += 1
            else:
                win.append(r)
        while len(win) < kmax and cursor < n and arrival[cursor] <= t:
            r = cursor
            cursor += 1
            if t + a[0] + w[0] * bins_of_dist[dist[r]] > arrival[r] + slo:
                drop += 1
            else:
                win.append(r)
        carry = []
        if not win:
            continue
        best, bestc = 0, -1
        for k in range(1, len(win) + 1):
            M = max(bins_of_dist[dist[r]] for r in win[:k])
            cnt = sum(1 for r in win[:k] if t + a[k - 1] + w[k - 1] * M <= arrival[r] + slo)
            if cnt > bestc:
                best, bestc = k, cnt
        k = best
        m = max(int(tb[r]) for r in win[:k])
        dur = int(a[k - 1] + w[k - 1] * m)
        for r in win[:k]:
            if t + dur <= arrival[r] + slo:
                fin += 1
            else:
                late += 1
        bat += 1
        busy += dur
        t += dur
        carry = win[k:]
    return [n, fin, drop, late, bat, busy, (t - int(arrival[0])) if n else 0]


def test_point_mass_replay_equals_planner():
    tf = gen.c5_trace_family("static")
    off, arr, dist, tb, slo = _small_trace(tf, S=8, n=300)
    F = oracle.cdf(tf.fam.counts)
    r = oracle.replay(F, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo)
    bins_of_dist = [int(np.argmax(row)) + 1 for row in tf.fam.counts]
    for s in range(len(slo)):
        sl = slice(off[s], off[s + 1])
        exp = _planner_replay(bins_of_dist, tf.profile.a, tf.profile.w, tf.profile.kmax,
                              arr[sl], dist[sl], tb[sl], int(slo[s]))
        assert r["counters"][s].tolist() == exp


def test_replay_empty_and_single():
    counts = np.zeros((1, 8), np.uint32)
    counts[0, 3] = 1
    F = oracle.cdf(counts)
    a, w = np.zeros(4, np.int64), np.arange(1, 5, dtype=np.int64)
    off = np.array([0, 0, 1], np.int64)
    r = oracle.replay(F, a, w, off, np.array([5], np.int64), np.array([0], np.int32), np.array([4], np.int16),
                      np.array([10, 10], np.int64), want_log=True)
    assert r["counters"][0].tolist() == [0] * 7
    assert r["counters"][1].tolist() == [1, 1, 0, 0, 1, 4, 4]
    assert r["log"].tolist() == [0, 1, 0]


# ---------------------------------------------------------------------------
# replay policy variants
# ---------------------------------------------------------------------------
import _policy_cases  # noqa: E402


@pytest.mark.parametrize("case", _policy_cases.load(), ids=lambda c: c["name"])
def test_policy_golden(case):
    x = _policy_cases.arrays(case)
    F = oracle.cdf(x["counts"])
    for key, exp in case["expect"].items():
        objective, drop = key.split("/")
        r = oracle.replay(F, x["a"], x["w"], x["off"], x["arrival"], x["dist"], x["tb"], x["slo"],
                          objective=objective, drop=drop, counts=x["counts"])
        assert dict(zip(oracle.COUNTER_FIELDS, r["counters"][0].tolist())) == exp, key


def test_expected_latency_thresholds_exact():
    """policy.expected_latency_thresholds implements t + a_1 + w_1 E[bin] > D_r
    exactly: check the equivalence D - t < thr  <=>  (D - t - a_1) total <
    w_1 sum_i i c_i (exact rationals) around every threshold."""
    from paper_2209_00159_b200 import policy
    rng = np.random.default_rng(5)
    for _ in range(50):
        B = int(rng.integers(4, 65))
        counts = rng.integers(0, 1000, (3, B)).astype(np.uint32)
        counts[:, -1] += 1
        a = np.array([int(rng.integers(0, 5000))], np.int64)
        w = np.array([int(rng.integers(1, 3000))], np.int64)
        thr = policy.expected_latency_thresholds(counts, a, w)
        for d in range(3):
            num = sum((i + 1) * int(c) for i, c in enumerate(counts[d]))
            den = int(counts[d].sum())
            for slack in range(int(thr[d]) - 3, int(thr[d]) + 3):
                assert (slack < thr[d]) == ((slack - int(a[0])) * den < int(w[0]) * num)
        assert (policy.hopeless_thresholds(counts, a, w) == a[0] + w[0] * (np.argmax(counts > 0, 1) + 1)).all()


@pytest.mark.parametrize("fam", ["skipnet", "gpt"])
def test_policy_invariants(fam):
    tf = gen.c5_trace_family(fam)
    off, arr, dist, tb, slo = _small_trace(tf, S=8, n=1500)
    F = oracle.cdf(tf.fam.counts)
    for objective in ("expected_finish", "finish_rate"):
        for drop in ("hopeless", "expected_latency"):
            r = oracle.replay(F, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo, want_log=True,
                              objective=objective, drop=drop, counts=tf.fam.counts)
            c = r["counters"]
            assert (c[:, 1] + c[:, 2] + c[:, 3] == c[:, 0]).all()
            r2 = oracle.replay(F, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo, follow_log=r["log"],
                               objective=objective, drop=drop, counts=tf.fam.counts)
            assert (r2["counters"] == c).all() and (r2["ties"][:, 2] == -1).all()
    # the expected-latency rule drops at least what the hopeless rule drops
    h = oracle.replay(F, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo)["counters"]
    e = oracle.replay(F, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo, drop="expected_latency",
                      counts=tf.fam.counts)["counters"]
    assert e[:, 2].sum() >= h[:, 2].sum()
