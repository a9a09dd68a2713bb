"""Oracle pins: closed forms, textbook reductions and invariants.

* Eq. 6: i.i.d. members => CDF of the max is F^k.
  Discrete uniform over B bins: G_k[i] = (i/B)^k.
* Geometric h_i ~ q^(i-1), q = 1/2, B = 4: F = 8/15, 4/5, 14/15, 1 and
  G_2 = 64/225, 16/25, 196/225, 1 (exact rationals).
* Mixed uniforms (member j uniform on bins 1..B_j): G_k[i] = prod_j min(1, i/B_j).
* Point masses reduce to the textbook constant-latency planner:
  E_k = #{r <= k : now + a_k + w_k * M_k <= D_r}, M_k the largest member bin.
* Eq. 5 for the uniform: E[max bin] = sum_i i((i/B)^k - ((i-1)/B)^k), and
  SPEC S:84 (c0 = 1, c1 = 0.5, k = 2, uniform on [0, 10]) -> 7.667 as B grows.
* Invariants: P in [0, 1]; P_r(k+1) <= P_r(k) for a monotone profile;
  E_k <= k; E_1 = P_1(1); E_k = sum_r P_r(k).

To read P_r(k) at a chosen bin i the tests put sigma_r = a_k + w_k * i + j with
0 <= j < w_k (the bin the batch finishes in); that choice is checked against
the brute-force enumerator in test_oracle_bruteforce.py, which tests the
deadline directly instead.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle


def _P(r, k):
    return k * (k - 1) // 2 + r


def test_cdf_values():
    F = oracle.cdf(np.array([[8, 4, 2, 1], [3, 1, 0, 0], [0, 0, 0, 5]], np.uint32))
    assert F[0].tolist() == [8 / 15, 12 / 15, 14 / 15, 1.0]
    assert F[1].tolist() == [0.75, 1.0, 1.0, 1.0]      # SPEC S:57 at the bin edge
    assert F[2].tolist() == [0.0, 0.0, 0.0, 1.0]


@pytest.mark.parametrize("B,k", [(4, 1), (8, 3), (16, 5), (64, 8), (256, 4)])
def test_iid_uniform_power(B, k):
    counts = np.full((1, B), 1 << 10, np.uint32)
    F = oracle.cdf(counts)
    a = np.full(k, 7, np.int64)
    w = np.arange(1, k + 1, dtype=np.int64) * 3
    rng = np.random.default_rng(B * 100 + k)
    for i in rng.choice(np.arange(0, B + 1), size=min(B + 1, 12), replace=False):
        sig = a[k - 1] + w[k - 1] * int(i) + int(rng.integers(0, w[k - 1]))
        dl = np.full(k, sig, np.int64)
        r = oracle.score(F, a, w, [0, k], dl, np.zeros(k, np.int32), [0], want_P=True)
        assert r["P"][0][_P(0, k)] == pytest.approx((i / B) ** k, abs=1e-15)


def test_geometric_exact():
    counts = np.array([[8, 4, 2, 1]], np.uint32)
    F = oracle.cdf(counts)
    expect = [Fraction(64, 225), Fraction(16, 25), Fraction(196, 225), Fraction(1)]
    a, w = np.array([0, 0]), np.array([1, 1])
    for i, e in enumerate(expect, start=1):
        r = oracle.score(F, a, w, [0, 2], [i, i], [0, 0], [0], want_P=True)
        assert r["P"][0][_P(0, 2)] == pytest.approx(float(e), abs=1e-15)
    # sigma below every bin -> P = 0 exactly; beyond B -> 1 exactly (A12)
    r = oracle.score(F, a, w, [0, 2], [0, 99], [0, 0], [0], want_P=True)
    assert r["P"][0][_P(0, 2)] == 0.0 and r["P"][0][_P(1, 2)] == 1.0


def test_mixed_uniforms():
    B = 12
    Bj = [3, 6, 12, 4]
    counts = np.zeros((len(Bj), B), np.uint32)
    for d, b in enumerate(Bj):
        counts[d, :b] = 5
    F = oracle.cdf(counts)
    k = len(Bj)
    a, w = np.zeros(k, np.int64), np.ones(k, np.int64)
    for i in range(0, B + 1):
        r = oracle.score(F, a, w, [0, k], np.full(k, i), np.arange(k), [0], want_P=True)
        expect = np.prod([min(1.0, i / b) for b in Bj])
        assert r["P"][0][_P(0, k)] == pytest.approx(expect, abs=1e-15)


def _planner(bins_of_dist, dist, deadline, now, a, w, kmax):
    """Textbook constant-latency planner: every member's time is known exactly."""
    K = min(len(dist), kmax)
    E = []
    for k in range(1, K + 1):
        M = max(bins_of_dist[d] for d in dist[:k])
        dur = a[k - 1] + w[k - 1] * M
        E.append(sum(1 for r in range(k) if now + dur <= deadline[r]))
    return E


def test_point_mass_is_constant_latency_planner():
    B = 32
    bins_of_dist = [16, 10, 1, 32]
    counts = np.zeros((4, B), np.uint32)
    for d, b in enumerate(bins_of_dist):
        counts[d, b - 1] = 1 << 30
    F = oracle.cdf(counts)
    rng = np.random.default_rng(4)
    kmax = 32
    a = np.full(kmax, 4000, np.int64)
    w = 250 * np.arange(1, kmax + 1, dtype=np.int64)
    for trial in range(60):
        n = int(rng.integers(0, 40))
        now = int(rng.integers(0, 1 << 40))
        dl = np.sort(now + rng.integers(-5000, 300000, n)).astype(np.int64)
        dist = rng.integers(0, 4, n).astype(np.int32)
        r = oracle.score(F, a, w, [0, n], dl, dist, [now], want_P=True)
        expect = _planner(bins_of_dist, dist, dl, now, a, w, kmax)
        K = min(n, kmax)
        assert r["E"][0][:K].tolist() == [float(e) for e in expect]
        assert set(np.unique(r["P"][0])) <= {0.0, 1.0}
        if K:
            best = max(expect)
            assert r["best_k"][0] == expect.index(best) + 1
        else:
            assert r["best_k"][0] == 0


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_expected_batch_latency_uniform(k):
    B = 50
    counts = np.full((1, B), 3, np.uint32)
    F = oracle.cdf(counts)
    a = np.full(k, 11, np.int64)
    w = 2 * np.arange(1, k + 1, dtype=np.int64)
    r = oracle.score(F, a, w, [0, k], np.zeros(k, np.int64), np.zeros(k, np.int32), [0], want_EL=True)
    emax = sum(i * ((i / B) ** k - ((i - 1) / B) ** k) for i in range(1, B + 1))
    assert r["EL"][0][k - 1] == pytest.approx(11 + w[k - 1] * emax, rel=1e-13)


def test_spec_s84_limit():
    """c0 = 1, c1 = 0.5, k = 2, uniform on [0, 10] -> 1 + 0.5*2*(20/3)
    = 7.667.  Units: 1 ms = 1000 ticks, B = 1000 bins of 10 ticks; the grid is
    discrete at upper edges, so the limit is approached within O(Delta)."""
    B, delta = 1000, 10
    counts = np.full((1, B), 1, np.uint32)
    F = oracle.cdf(counts)
    a = np.array([1000, 1000], np.int64)
    w = np.array([round(0.5 * 1 * delta), round(0.5 * 2 * delta)], np.int64)
    r = oracle.score(F, a, w, [0, 2], [0, 0], [0, 0], [0], want_EL=True)
    assert r["EL"][0][1] / 1000 == pytest.approx(7.667, abs=0.01)


def test_invariants_random():
    rng = np.random.default_rng(7)
    D, B, kmax = 6, 24, 20
    counts = rng.integers(0, 5, (D, B)).astype(np.uint32)
    counts[:, -1] += 1
    F = oracle.cdf(counts)
    a = np.cumsum(rng.integers(0, 3, kmax)).astype(np.int64) + 5
    w = np.cumsum(rng.integers(0, 2, kmax)).astype(np.int64) + 1
    Q = 200
    lens = rng.integers(0, 30, Q)
    off = np.concatenate([[0], np.cumsum(lens)])
    now = rng.integers(0, 1 << 40, Q)
    dl = np.concatenate([np.sort(now[q] + rng.integers(-10, 400, lens[q])) for q in range(Q)]).astype(np.int64)
    dist = rng.integers(0, D, off[-1]).astype(np.int32)
    r = oracle.score(F, a, w, off, dl, dist, now, want_P=True)
    E, P = r["E"], r["P"]
    assert (P >= 0).all() and (P <= 1).all()
    for q in range(Q):
        K = min(lens[q], kmax)
        assert (E[q][K:] == 0).all()
        for k in range(1, K + 1):
            row = P[q][_P(0, k):_P(0, k) + k]
            assert E[q][k - 1] == pytest.approx(row.sum(), abs=1e-12)
            assert E[q][k - 1] <= k + 1e-12
            if k < K:
                nxt = P[q][_P(0, k + 1):_P(0, k + 1) + k]
                assert (nxt <= row + 1e-15).all()       # P_r(k+1) <= P_r(k)
        if K:
            assert E[q][0] == P[q][0]
            assert r["best_k"][q] == int(np.argmax(E[q][:K])) + 1
            assert r["best_E"][q] == E[q][r["best_k"][q] - 1]
        else:
            assert r["best_k"][q] == 0
