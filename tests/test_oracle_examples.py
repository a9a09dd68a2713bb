"""Oracle pins: exact worked examples (golden fixtures with citations).

Appendix A (tests/golden/appendix_a.json), derived by hand from the model
(Eq. 3-4 :479-491, product form of Eq. 6/8 :503-535):
B = 4, tau_i = i, t = 0, a = [0, 1, 1], w = [1, 1, 2] so the k-batch whose
slowest member sits in bin m runs dur_1 = m, dur_2 = 1 + m, dur_3 = 1 + 2m.

Ex1  (6, 1/2@1 1/2@4), (9, 1@2), (12, uniform):
     k=1: dur = X1 <= 4 <= 6 -> P = 1, E_1 = 1.
     k=2: dur = 1 + max(X1, 2) in {3, 5}, both <= 6 and <= 9 -> E_2 = 2.
     k=3: dur = 1 + 2M; r1 needs M <= 2: Pr = 1/2 * 1 * 2/4 = 1/4;
          r2 needs M <= 4 -> 1; r3 needs M <= 5.5 -> 1.  E_3 = 9/4, k* = 3.
Ex2  (5, 1@2), (8, uniform), (11, uniform):
     E_1 = 1; k=2: dur = 1 + max(2, X2) <= 5 -> E_2 = 2;
     k=3: r1 M <= 2: 1 * 2/4 * 2/4 = 1/4; r2 M <= 3: (3/4)^2 = 9/16; r3 -> 1.
     E_3 = 29/16 < 2 -> k* = 2 (interior argmax).
Ex3  (2, 1/2@2 1/2@3), (3, 1/2@1 1/2@4), (8, 1@2):
     k=1: X1 <= 2 -> 1/2.  k=2: r1 needs M <= 1 -> 0; r2 M <= 2 -> 1/2*1/2 = 1/4.
     k=3: r1 M <= 0 -> 0; r2 M <= 1 -> 0; r3 M <= 3 -> 1 * 1/2 * 1 = 1/2.
     E = [1/2, 1/4, 1/2]: exact tie, smallest k wins -> k* = 1.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("ex", _load("appendix_a.json")["examples"], ids=lambda e: e["name"])
def test_appendix_a(ex):
    g = _load("appendix_a.json")
    counts = np.array(ex["counts"], np.uint32)
    F = oracle.cdf(counts)
    K = len(ex["deadline"])
    r = oracle.score(F, g["a"], g["w"], [0, K], ex["deadline"], np.arange(K), [g["now"]], want_P=True)
    E = [float(Fraction(x)) for x in ex["E"]]
    assert np.allclose(r["E"][0], E, rtol=0, atol=1e-15)
    assert r["best_k"][0] == ex["k_star"]
    P3 = [float(Fraction(x)) for x in ex["P_k3"]]
    assert np.allclose(r["P"][0][3:6], P3, rtol=0, atol=1e-15)
    # the brute-force enumerator agrees
    Pb, Eb = oracle.bruteforce(counts, g["a"], g["w"], ex["deadline"], np.arange(K), g["now"])
    assert np.allclose(Eb, E, atol=1e-15)
    assert np.allclose(Pb[3:6], P3, atol=1e-15)


def _spec_trace(case):
    B = 100
    # dist 0: point mass at 10 ms, dist 1: point mass at 100 ms
    # dist 2: 1/2 at 10 ms, 1/2 at 100 ms
    counts = np.zeros((3, B), np.uint32)
    counts[0, 9] = 1
    counts[1, 99] = 1
    counts[2, 9] = counts[2, 99] = 1
    dist = np.array(case.get("dist", [0 if x == 10 else 1 for x in case["true_ms"]]), np.int32)
    tb = np.array(case["true_ms"], np.int16)
    kmax = 4
    a = np.zeros(kmax, np.int64)
    w = np.arange(1, kmax + 1, dtype=np.int64)
    n = len(dist)
    return counts, a, w, np.array([0, n], np.int64), np.array(case["arrival"], np.int64), dist, tb, \
        np.array([case["slo"]], np.int64)


@pytest.mark.parametrize("case", _load("spec_replay.json")["cases"], ids=lambda c: c["name"])
def test_spec_replay(case):
    counts, a, w, off, arr, dist, tb, slo = _spec_trace(case)
    r = oracle.replay(oracle.cdf(counts), a, w, off, arr, dist, tb, slo, want_log=True)
    got = dict(zip(oracle.COUNTER_FIELDS, r["counters"][0].tolist()))
    assert got == case["expect"]
    c = r["counters"][0]
    assert c[1] + c[2] + c[3] == c[0]          # conservation


def test_spec_replay_decisions():
    """S:430 order A: at t=0 E = [1, 2, 0, 0] -> k*=2 (dur 20); at t=20 the
    100-ms pair has sigma 130: E = [1, 0] -> k*=1 (dur 100, ends 120); the last
    request has sigma 30 < 100 -> hopeless, dropped."""
    case = _load("spec_replay.json")["cases"][1]
    counts, a, w, off, arr, dist, tb, slo = _spec_trace(case)
    r = oracle.replay(oracle.cdf(counts), a, w, off, arr, dist, tb, slo, want_log=True)
    assert r["log"].tolist()[:3] == [2, 1, 0]


def test_spec_batch_latency_examples():
    """SPEC S:82-83 (batch_latency): c0=0, c1*k=1 is the identity (the paper's
    toy example 'no overhead for batching'); c0=2, c1=1, k=3 on a
    point mass at 10 gives a point mass at 32 (expectation 32)."""
    B = 16
    counts = np.zeros((1, B), np.uint32)
    counts[0, 9] = 7                      # point mass at tau_10 = 10
    F = oracle.cdf(counts)
    a = np.array([2, 2, 2], np.int64)
    w = np.array([1, 2, 3], np.int64)     # c1 * k * Delta, Delta = 1
    for sigma, expect in [(31, 0.0), (32, 1.0), (40, 1.0)]:
        r = oracle.score(F, a, w, [0, 3], [sigma] * 3, [0, 0, 0], [0], want_P=True, want_EL=True)
        assert r["P"][0][3] == expect     # P_1(3)
        assert r["EL"][0][2] == 32.0
    # identity: a = 0, w = 1 for k = 2 -> P_r(2) = Pr(max <= sigma)
    counts2 = np.array([[1, 0, 0, 1], [0, 0, 1, 0]], np.uint32)
    r = oracle.score(oracle.cdf(counts2), [0, 0], [1, 1], [0, 2], [3, 4], [0, 1], [0], want_P=True)
    assert r["P"][0][1] == 0.5 and r["P"][0][2] == 1.0


def test_spec_max_order_examples():
    """two equal-mass point-like bins at 10 and 100, k=2 -> CDF of the
    max at 10+ is (1/2)^2 = 0.25 (enumeration of 4 outcomes).  S:74: point masses
    at 5 and 50 -> the max is the point mass at 50."""
    B = 100
    counts = np.zeros((3, B), np.uint32)
    counts[0, 9] = counts[0, 99] = 1
    counts[1, 4] = 1
    counts[2, 49] = 1
    F = oracle.cdf(counts)
    a, w = [0, 0], [1, 1]
    r = oracle.score(F, a, w, [0, 2], [10, 10], [0, 0], [0], want_P=True)
    assert r["P"][0][1] == 0.25
    r = oracle.score(F, a, w, [0, 2], [49, 50], [1, 2], [0], want_P=True)
    assert r["P"][0][1] == 0.0 and r["P"][0][2] == 1.0


def test_cold_start():
    """total == 0 is the cold-start error."""
    with pytest.raises(oracle.OracleError):
        oracle.cdf(np.zeros((1, 4), np.uint32))
