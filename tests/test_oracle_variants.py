"""Pins of oracle/variants.py against independent
results:
* edge bins + the Eq. 3 table + one unit step == the O1 oracle (oracle.c);
* uniform bins: i.i.d. uniform histograms with the identity grid give the
  continuous closed form P(max <= u) = (u / B)^k; SPEC S:55-57 CDF examples;
  Monte Carlo over members drawn uniformly within their bins;
* log-spaced grids: brute-force enumeration of joint bin outcomes with the
  table's durations;
* step costs: brute force over joint outcomes of the credit c_last - cost(finish)
  computed from the multi-step cost function itself."""
import itertools
import math

import numpy as np

import gen
import oracle
from oracle import variants as va


def _eq3_table(a, w, B):
    m = np.arange(B + 1, dtype=np.int64)
    return np.asarray(a, np.int64)[:, None] + np.asarray(w, np.int64)[:, None] * m[None, :]


def test_edge_eq3_unit_step_is_o1():
    c = gen.config2(Q=24, n=12, kmax=8)
    q = c.queues
    dur = _eq3_table(c.profile.a, c.profile.w, c.fam.B)
    E, best = va.score(c.fam.counts, dur, q.offsets, q.deadline, q.dist, q.now)
    ref = oracle.score(oracle.cdf(c.fam.counts), c.profile.a, c.profile.w, q.offsets, q.deadline, q.dist, q.now)
    assert np.abs(E - ref["E"]).max() < 1e-12
    assert (best == ref["best_k"]).all()


def test_uniform_bins_iid_closed_form():
    B = 8
    counts = np.ones((3, B), np.int64)  # every app uniform over the bins
    dur = np.tile(np.arange(B + 1, dtype=np.int64) * 10, (4, 1))  # position m -> 10 m ticks
    F = va.cdf_rows(counts)
    for k in (1, 2, 4):
        for x in (0, 7, 10, 33, 55, 79, 80, 200):
            got = va.finish_prob(F, [0, 1, 2, 0][:k], dur[k - 1], x, True)
            assert abs(got - min(1.0, x / 80.0) ** k) < 1e-14, (k, x, got)


def test_uniform_bins_spec_cdf_examples():
    # S:55-57 on a single member: bin (10, 20] holding all mass -> F(15) = 0.5, F(20) = 1;
    # two bins (0,10]: 3, (10,20]: 1 -> F(10) = 0.75
    dur = np.array([[0, 10, 20]], np.int64)
    F1 = va.cdf_rows(np.array([[0, 1]]))
    assert va.finish_prob(F1, [0], dur[0], 15, True) == 0.5
    assert va.finish_prob(F1, [0], dur[0], 20, True) == 1.0
    F2 = va.cdf_rows(np.array([[3, 1]]))
    assert va.finish_prob(F2, [0], dur[0], 10, True) == 0.75


def test_uniform_bins_monte_carlo():
    rng = np.random.default_rng(gen.SEED_BASE + 940)
    counts = rng.integers(1, 20, size=(3, 6))
    log_grid = np.round(100 * 2.0 ** (np.arange(7) / 2.0)).astype(np.int64)  # log-spaced positions
    F = va.cdf_rows(counts)
    pm = counts / counts.sum(axis=1, keepdims=True)
    dists = [0, 2, 1]
    n = 400_000
    pos = np.zeros(n)
    for d in dists:
        b = rng.choice(6, size=n, p=pm[d])
        pos = np.maximum(pos, b + rng.random(n))  # uniform within bin b+1 = (b, b+1]
    dur_of = np.interp(pos, np.arange(7), log_grid)  # duration linear between grid positions
    for x in (150, 260, 420, 700, 900):
        est = (dur_of <= x).mean()
        got = va.finish_prob(F, dists, log_grid, x, True)
        assert abs(got - est) <= 5 * math.sqrt(max(est * (1 - est), 1e-12) / n) + 1e-12, (x, got, est)


def test_log_grid_edge_bruteforce():
    rng = np.random.default_rng(gen.SEED_BASE + 941)
    B = 5
    counts = rng.integers(0, 6, size=(4, B))
    counts[:, 0] += 1
    tab = np.round(50 * 1.7 ** np.arange(B + 1)).astype(np.int64)
    dur = np.stack([tab + 7 * k for k in range(3)])
    pm = counts / counts.sum(axis=1, keepdims=True)
    F = va.cdf_rows(counts)
    dists = [3, 0, 2]
    for k in (1, 2, 3):
        for x in (40, 60, 100, 160, 300, 600):
            want = 0.0
            for bins in itertools.product(range(B), repeat=k):
                pr = math.prod(pm[dists[j], bins[j]] for j in range(k))
                if dur[k - 1][max(bins) + 1] <= x:  # mass of bin b at its upper edge, position b+1
                    want += pr
            assert abs(va.finish_prob(F, dists[:k], dur[k - 1], x, False) - want) < 1e-14


def test_step_costs_bruteforce_credit():
    rng = np.random.default_rng(gen.SEED_BASE + 942)
    B = 4
    counts = rng.integers(1, 5, size=(3, B))
    pm = counts / counts.sum(axis=1, keepdims=True)
    dur = _eq3_table([5, 6, 8], [10, 12, 13], B)
    offs, costs = [-5, 0, 20], [0.5, 1.5, 2.0]
    dl = np.array([30, 41, 55], np.int64)
    dist = np.array([0, 2, 1], np.int32)
    E, _ = va.score(counts, dur, np.array([0, 3]), dl, dist, np.array([0]), step_offsets=offs, step_costs=costs)

    def cost(finish, D):  # the multi-step cost function: c_s once the s-th deadline is missed
        c = 0.0
        for o, cs in zip(offs, costs):
            if finish > D + o:
                c = cs
        return c

    for k in (1, 2, 3):
        want = 0.0
        for bins in itertools.product(range(B), repeat=k):
            pr = math.prod(pm[dist[j], bins[j]] for j in range(k))
            finish = dur[k - 1][max(bins) + 1]
            want += pr * sum(costs[-1] - cost(finish, dl[r]) for r in range(k))
        assert abs(E[0, k - 1] - want) < 1e-12, (k, E[0, k - 1], want)
