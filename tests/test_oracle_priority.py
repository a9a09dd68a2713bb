"""Pins of oracle/priority.py (Eq. 1-2 priority, batch latency of a mixture,
PopBatch) against what the paper and the mathematics fix, independent of the
oracle's own formulas:

* the batch-latency pmf against brute-force enumeration of every bs-tuple of
  (application, bin) draws (Eq. 6 with a mixture);
* log p against Eq. 1 evaluated from its DEFINITION, p = (E[C_delay] -
  E[C_now]) / E[L] with C = 1[t > D], tau ~ Exp(b): by numerical
  quadrature of the convolution P(tau + L <= sigma) and by Monte Carlo;
* E[L] against the quadrature of the survival function;
* the limits b -> 0 (p -> P(L <= sigma) / E[L]) and the milestone form
  p(t) = alpha e^{bt} + beta between milestones;
* PopBatch against the order invariants of "the bs highest priorities";
* the piecewise-step cost against Eq. 1 with the multi-step
  cost function itself, by quadrature.
"""
import itertools
import math

import numpy as np
import pytest
from scipy import integrate

import gen
from oracle import priority as pr


def _fam():
    rng = np.random.default_rng(gen.SEED_BASE + 901)
    D, B = 3, 6
    counts = rng.integers(0, 9, size=(D, B))
    counts[:, 2] += 1  # every row has a positive total
    return counts


def _F_L(pm, a, w):
    """Piecewise-linear CDF of L with pm spread uniformly over (a + w(i-1), a + w i]."""
    edges = a + w * np.arange(len(pm) + 1, dtype=np.float64)
    G = np.concatenate([[0.0], np.cumsum(pm)])
    return lambda x: float(np.interp(x, edges, G, left=0.0, right=1.0)), edges


@pytest.mark.parametrize("bs", [1, 2, 3])
def test_batch_pmf_bruteforce(bs):
    counts = _fam()
    D, B = counts.shape
    wts = np.array([1.0, 2.0, 0.5])
    p_draw = (wts[:, None] * counts / counts.sum(axis=1, keepdims=True)) / wts.sum()  # P(app d, bin i)
    pm = np.zeros(B)
    cells = [(d, i) for d in range(D) for i in range(B)]
    for tup in itertools.product(cells, repeat=bs):
        pm[max(i for _, i in tup)] += math.prod(p_draw[d, i] for d, i in tup)
    got = pr.batch_latency_pmf(counts, bs, wts)
    assert np.allclose(got, pm, rtol=0, atol=1e-14)
    assert abs(got.sum() - 1.0) < 1e-14


@pytest.mark.parametrize("bs,b", [(1, 1e-3), (2, 2e-2), (3, 3e-4)])
def test_priority_matches_eq1_definition_quadrature(bs, b):
    counts = _fam()
    a, w = 250.0, 100.0
    pm = pr.batch_latency_pmf(counts, bs)
    F, edges = _F_L(pm, a, w)
    EL_quad = integrate.quad(lambda x: 1.0 - F(x), 0.0, edges[-1], points=list(edges), limit=200)[0]
    assert abs(pr.expected_latency(pm, a, w) - EL_quad) < 1e-9 * EL_quad
    sig = np.array([-50.0, 0.0, a - 1, a, a + 37.0, a + w, a + 2.5 * w, a + 4 * w + 1, edges[-1], edges[-1] + 300.0])
    got = pr.log_priority(pm, a, w, b, sig)
    for s, lp in zip(sig, got):
        # E[C_delay] - E[C_now] = P(t + tau + L > D) - P(t + L > D) = F_L(sigma) - P(tau + L <= sigma)
        if s <= 0:
            conv = 0.0
        else:
            pts = [s - e for e in edges if 0 < s - e < s]
            conv = integrate.quad(lambda u: b * math.exp(-b * u) * F(s - u), 0.0, s, points=pts or None,
                                  limit=400, epsabs=1e-15, epsrel=1e-12)[0]
        p_def = (F(s) - conv) / EL_quad
        if p_def <= 1e-300:
            assert lp == -np.inf
        else:
            assert abs(math.exp(lp) - p_def) <= 1e-9 * p_def + 1e-15, (s, math.exp(lp), p_def)


def test_priority_monte_carlo():
    counts = _fam()
    a, w, b, bs = 250.0, 100.0, 4e-3, 2
    pm = pr.batch_latency_pmf(counts, bs)
    rng = np.random.default_rng(gen.SEED_BASE + 902)
    n = 2_000_000
    i = rng.choice(len(pm), size=n, p=pm / pm.sum())
    L = a + w * (i + rng.random(n))
    tau = rng.exponential(1.0 / b, size=n)
    EL = L.mean()
    for s in (a + 1.5 * w, a + 3.2 * w, a + 7 * w):
        x = ((L <= s) & (tau + L > s)).astype(np.float64)
        est, se = x.mean() / EL, x.std() / math.sqrt(n) / EL
        p = math.exp(pr.log_priority(pm, a, w, b, [s])[0])
        assert abs(p - est) <= 5 * se + 1e-4 * p


def test_small_b_limit_and_milestone_form():
    counts = _fam()
    a, w, bs = 250.0, 100.0, 3
    pm = pr.batch_latency_pmf(counts, bs)
    F, edges = _F_L(pm, a, w)
    EL = pr.expected_latency(pm, a, w)
    b = 1e-10
    for s in (a + 0.5 * w, a + 2 * w, edges[-1] + 10):
        p = math.exp(pr.log_priority(pm, a, w, b, [s])[0])
        # b -> 0: tau -> infinity, E[C_delay] -> 1, p -> F_L(sigma) / E[L]
        assert abs(p - F(s) / EL) <= 1e-6 * F(s) / EL
    # beyond the last milestone (sigma >= a + wB) only full bins remain:
    # p(t) = alpha e^{bt}, i.e. p(sigma + d) = p(sigma) e^{-bd}
    b = 2e-3
    s0 = edges[-1] + 5
    l0, l1 = pr.log_priority(pm, a, w, b, [s0, s0 + 321.0])
    assert abs((l1 - l0) + b * 321.0) < 1e-12
    # between two milestones inside bin i the form is alpha e^{bt} + beta: second
    # differences of p in t obey p'' = b p' (no other terms)
    s = a + 2 * w + np.array([20.0, 40.0, 60.0])
    p = np.exp(pr.log_priority(pm, a, w, b, s))
    # t = D - sigma: in t, p = alpha e^{bt} + beta with equally spaced t -> geometric differences
    d1, d2 = p[1] - p[0], p[2] - p[1]
    assert abs(d1 / d2 - math.exp(b * 20.0)) < 1e-9


def test_priority_zero_before_any_outcome():
    counts = _fam()
    counts[:, :2] = 0
    pm = pr.batch_latency_pmf(counts, 2)
    a, w = 100.0, 50.0
    got = pr.log_priority(pm, a, w, 1e-3, [a + 2 * w, a + 2 * w + 1])
    assert got[0] == -np.inf and np.isfinite(got[1])


def test_pop_batch_invariants():
    rng = np.random.default_rng(gen.SEED_BASE + 903)
    for trial in range(200):
        n, S = int(rng.integers(0, 300)), 4
        v = rng.integers(-5, 5, size=(n, S)).astype(np.float32)
        v[rng.random((n, S)) < 0.15] = -np.inf
        v[rng.random((n, S)) < 0.05] = np.nan
        bs = int(rng.integers(0, 6))
        sel = pr.pop_batch(v, bs, S)
        if not 1 <= bs <= S:
            assert sel == []
            continue
        col = v[:256, bs - 1]
        ok = [r for r in range(len(col)) if np.isfinite(col[r])]
        assert len(sel) == min(bs, len(ok)) and len(set(sel)) == len(sel)
        assert all(r in ok for r in sel)
        rest = [r for r in ok if r not in sel]
        for j, r in enumerate(sel):
            if j:
                assert (col[sel[j - 1]], -sel[j - 1]) > (col[r], -r)
            for u in rest:  # every unselected candidate is lower, or equal and later
                assert (col[r], -r) > (col[u], -u)


def test_piecewise_step_cost_matches_definition():
    """Appendix: with a multi-step cost C(x) = c_s for finish
    times x in (D + off_s, D + off_{s+1}] (c_0 = 0 before the first deadline),
    Eq. 1's E[C_delay] - E[C_now] evaluated from that definition by quadrature
    equals the oracle's sum of single-step priorities."""
    counts = _fam()
    a, w, b, bs = 250.0, 100.0, 3e-3, 2
    offs, costs = [0.0, 150.0, 420.0], [1.0, 2.5, 3.0]
    pm = pr.batch_latency_pmf(counts, bs)
    F, edges = _F_L(pm, a, w)
    EL = pr.expected_latency(pm, a, w)

    def cdf_conv(y):  # P(tau + L <= y)
        if y <= 0:
            return 0.0
        pts = [y - e for e in edges if 0 < y - e < y]
        return integrate.quad(lambda u: b * math.exp(-b * u) * F(y - u), 0.0, y, points=pts or None, limit=400,
                              epsabs=1e-15, epsrel=1e-12)[0]

    def expected_cost(cdf, sigma):  # E[C] with finish time measured from now: x <= sigma + off_s is on time for s
        lv = [cdf(sigma + o) for o in offs]  # P(finish within deadline s)
        # cost c_{s} applies when finishing after deadline s but within deadline s+1 (c_last after the last)
        e = 0.0
        for s in range(len(offs)):
            p_after_s = 1.0 - lv[s]
            p_after_next = 1.0 - lv[s + 1] if s + 1 < len(offs) else 0.0
            e += costs[s] * (p_after_s - p_after_next)
        return e

    for s in (a + 0.5 * w, a + 2.3 * w, a + 5 * w, edges[-1] + 100, edges[-1] + 600):
        p_def = (expected_cost(cdf_conv, s) - expected_cost(F, s)) / EL
        got = math.exp(pr.log_priority_steps(pm, a, w, b, [s], offs, costs)[0])
        assert abs(got - p_def) <= 1e-9 * p_def + 1e-15, (s, got, p_def)
    # one step with cost 1 at offset 0 is the single-step priority
    sig = np.array([a + 1.5 * w, a + 4 * w])
    assert np.array_equal(pr.log_priority_steps(pm, a, w, b, sig, [0.0], [1.0]), pr.log_priority(pm, a, w, b, sig))


@pytest.mark.parametrize("bs", [1, 8, 40])
def test_batch_logpmf_exact_rationals_beyond_fp64_range(bs):
    """log pm_i against exact rational arithmetic, including bin masses far
    below the fp64 range (F = 2^-20 in the first bin, bs = 40: G = 2^-800)."""
    from fractions import Fraction
    counts = np.array([[1, 0, 5, 1000, 2**20 - 1006], [0, 3, 0, 7, 2**20 - 10]], dtype=np.int64)
    T = 2**20
    Fmix = [(Fraction(int(counts[0, :i + 1].sum()), T) + Fraction(int(counts[1, :i + 1].sum()), T)) / 2
            for i in range(counts.shape[1])]
    G = [f ** bs for f in Fmix]
    got = pr.batch_latency_logpmf(counts, bs)
    prev = Fraction(0)
    for i, g in enumerate(G):
        pm = g - prev
        prev = g
        if pm == 0:
            assert got[i] == -np.inf
        else:
            want = math.log(pm.numerator) - math.log(pm.denominator)
            assert abs(got[i] - want) <= 1e-12 * max(1.0, abs(want)), (i, got[i], want)


# ---------------------------------------------------------------------------
# the store-format branch (store_fp32=True) and its distance to the exact model
# ---------------------------------------------------------------------------

def _rn_f32_of_log2(num: int, den: int):
    """fl32(log2(num/den)) by RN, decided in exact arithmetic: log2 to 60
    decimal digits (decimal module, independent of numpy's log2), then the
    nearest float32 among the candidates around it."""
    from decimal import Decimal, getcontext
    from fractions import Fraction
    getcontext().prec = 60
    if num == den:
        return np.float32(0.0), Fraction(1)       # log2 1 = 0 exactly
    x = (Decimal(num) / Decimal(den)).ln() / Decimal(2).ln()
    xf = Fraction(x)
    c = np.float32(float(x))
    cands = [c, np.nextafter(c, np.float32(-np.inf)), np.nextafter(c, np.float32(np.inf))]
    dist = [abs(Fraction(float(v)) - xf) for v in cands]
    best = cands[int(np.argmin(dist))]
    gap = sorted(dist)[1] - sorted(dist)[0]     # distance from a rounding midpoint (x2)
    return best, gap / abs(xf)


@pytest.mark.parametrize("seed", [0, 1])
def test_mixture_cdf_store_fp32_is_the_rounded_model(seed):
    """mixture_cdf(store_fp32=True) is the mixture of F^_d = 2^{RN32(log2 F_d)}
    (the store's data format, include/orloj.h): checked against the RN
    rounding decided in exact arithmetic and 2^x evaluated with 60-digit
    decimals, with weights, on rows with empty bins, near-1 CDFs (single-count
    tails at total 2^30, where the rounding erases masses) and exact powers
    of two (log2 F an integer)."""
    from decimal import Decimal, getcontext
    from fractions import Fraction
    getcontext().prec = 60
    rng = np.random.default_rng(gen.SEED_BASE + 930 + seed)
    D, B = 4, 12
    counts = np.zeros((D, B), np.int64)
    counts[0] = rng.integers(0, 50, B)
    counts[0, 3] += 1
    counts[1] = gen.largest_remainder(rng.dirichlet(np.ones(B)))        # total 2^30
    counts[2, :] = 0
    counts[2, 1], counts[2, 5], counts[2, 11] = 1 << 28, (1 << 30) - (1 << 28) - 3, 3   # F = 1/4 exactly; tails
    counts[3, 0], counts[3, B - 1] = (1 << 30) - 1, 1
    weights = [0.5, 2.0, 1.0, 0.25] if seed else None
    got = pr.mixture_cdf(counts, weights, store_fp32=True)
    wts = [Fraction(1)] * D if weights is None else [Fraction(x) for x in weights]
    cum = np.cumsum(counts, axis=1)
    tot = counts.sum(axis=1)
    for i in range(B):
        acc = Fraction(0)
        for d in range(D):
            if cum[d, i] == 0:
                continue                            # F = 0: log2 = -inf exactly, 2^-inf = 0
            x32, rel_gap = _rn_f32_of_log2(int(cum[d, i]), int(tot[d]))
            assert rel_gap > 2.0 ** -40, "too close to a rounding midpoint to decide"
            assert np.float32(np.log2(cum[d, i] / tot[d])) == x32      # numpy's path rounds the same way
            acc += wts[d] * Fraction(Decimal(2) ** Decimal(float(x32)))
        ref = acc / sum(wts)
        assert abs(got[i] - float(ref)) <= 4e-16 * float(ref) + 1e-300, (i, got[i], float(ref))
    # F = 1/4 exactly survives the rounding exactly; the tail masses of row 3 vanish
    assert pr.mixture_cdf(counts[2:3], store_fp32=True)[1] == 0.25
    F3 = pr.mixture_cdf(counts[3:4], store_fp32=True)
    assert F3[0] < 1.0 and F3[B - 1] == 1.0


def test_store_rounding_bound_holds():
    """The first-order bound on how far the store format moves log p from the
    exact histogram model (store_rounding_log_priority_bound) covers the
    actual difference between the two oracle branches on every workload
    family, batch size and slack.  Within e^10 of the size's largest priority
    it stays below 1e-2 (largest: the RDI-like family, a few 1e-3).  Far
    below that it grows and is infinite where p is decided by bins whose mass
    the rounding may erase (near-empty bins at the start of L_bs's support;
    RDI-like at b = 20 / mean: log p more than 20 below the maximum), which
    the tests report rather than bound."""
    fams = [("P1", gen.config_priority())] + [(f, gen.c5_trace_family(f)) for f in gen.C5_FAMILIES]
    for name, cfg in fams:
        counts, a, w = cfg.fam.counts, cfg.profile.a, cfg.profile.w
        for b in (0.05 / cfg.fam.mean_ticks(), 1.0 / cfg.fam.mean_ticks(), 20.0 / cfg.fam.mean_ticks()):
            for bs in (1, 2, 5, 16, 32):
                if bs > len(a):
                    continue
                ak, wk = float(a[bs - 1]), float(w[bs - 1])
                sig = np.linspace(-100.0, (ak + wk * counts.shape[1]) * 1.3, 1500)
                p0 = pr.log_priority_lp(pr.batch_latency_logpmf(counts, bs), ak, wk, b, sig)
                p1 = pr.log_priority_lp(pr.batch_latency_logpmf(counts, bs, store_fp32=True), ak, wk, b, sig)
                assert (np.isneginf(p0) == np.isneginf(p1)).all()
                fin = np.isfinite(p0)
                bound = pr.store_rounding_log_priority_bound(counts, ak, wk, b, sig, bs)
                relevant = fin & (p0 >= p0[fin].max() - 10.0)
                assert np.isfinite(bound[relevant]).all(), (name, bs, b)
                fb = fin & np.isfinite(bound)
                assert bound[relevant].max() < 1e-2, (name, bs)
                assert (np.abs(p0[fb] - p1[fb]) <= bound[fb]).all(), (name, bs, b)
