"""Oracle pin: brute-force enumeration of joint outcomes.

The enumerator walks every outcome (x_1..x_k) in {1..B}^k, accumulates the
probability of each value of the max, and tests the deadline itself
(now + a_k + w_k * m <= D_r) — it uses neither the product of CDFs nor the
floor lookup, so a dropped factor, a wrong index or an off-by-one in the
lookup of ``oracle.score`` fails here.
"""
import numpy as np
import pytest

import gen
import oracle


def _random_case(seed, n, B, D):
    rng = np.random.default_rng(seed)
    counts = np.stack([gen.largest_remainder(rng.dirichlet(np.ones(B) * 0.7)) for _ in range(D)])
    counts[rng.random((D, B)) < 0.2] = 0           # holes in the support
    counts[:, rng.integers(0, B, D)] += 1            # never empty
    a = np.cumsum(rng.integers(0, 3, n)).astype(np.int64)
    w = np.cumsum(rng.integers(0, 3, n)).astype(np.int64) + 1
    now = int(rng.integers(0, 1 << 40))
    dl = np.sort(now + rng.integers(0, int(a[-1] + w[-1] * B + 3), n)).astype(np.int64)
    dist = rng.integers(0, D, n).astype(np.int32)
    return counts.astype(np.uint32), a, w, now, dl, dist


@pytest.mark.parametrize("seed", range(6))
def test_bruteforce_matches_score(seed):
    counts, a, w, now, dl, dist = _random_case(seed, n=5, B=7, D=3)
    F = oracle.cdf(counts)
    n = len(dl)
    r = oracle.score(F, a, w, [0, n], dl, dist, [now], want_P=True)
    Pb, Eb = oracle.bruteforce(counts, a, w, dl, dist, now)
    assert np.abs(r["P"][0] - Pb).max() < 1e-13
    assert np.abs(r["E"][0] - Eb).max() < 1e-13


def test_bruteforce_config1():
    """C1 in full: 1 queue, 8 requests, 8 Dirichlet(1) pmfs over 16 bins,
    sum_k 16^k ~ 4.6e9 leaves."""
    c = gen.config1()
    q = c.queues
    F = oracle.cdf(c.fam.counts)
    r = oracle.score(F, c.profile.a, c.profile.w, q.offsets, q.deadline, q.dist, q.now, want_P=True)
    Pb, Eb = oracle.bruteforce(c.fam.counts, c.profile.a, c.profile.w, q.deadline, q.dist, int(q.now[0]))
    assert np.abs(r["P"][0] - Pb).max() < 1e-12
    assert np.abs(r["E"][0] - Eb).max() < 1e-12
    assert r["best_k"][0] == int(np.argmax(Eb)) + 1
