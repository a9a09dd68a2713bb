"""Oracle pin: the paper's Eq. 8 vs the product of CDFs.

Eq. 8 (Ozbey et al.) gives the PDF of the max of k independent, non-identical
variables as a signed sum over subsets s with the subset means F^s, f^s of
Eq. 7.  The oracle instead multiplies CDFs.  These tests tie
the two together without using the product on the Eq. 8 side:

1. ``eq8_pdf`` evaluates Eq. 8 literally; for power-law CDFs F_i(x) = x^alpha_i
   on [0, 1] its numerical integral equals prod_i F_i(x) (= x^sum alpha).
2. Integrating Eq. 8 term by term gives sum_kappa (-1)^(k-kappa) kappa^k/k!
   sum_{|s|=kappa} [F^s]^k; with exact rationals that equals prod F_i exactly.
3. The oracle's G_k (read through P_r(k)) equals the integrated Eq. 8 on
   random histograms.
4. With all members identical Eq. 8 collapses to Eq. 6's k F^(k-1) f.
"""
from fractions import Fraction

import numpy as np
import pytest
from scipy.integrate import quad

import oracle


@pytest.mark.parametrize("alphas", [(1.0, 2.0), (0.5, 1.5, 3.0), (1.0, 1.0, 2.0, 0.7), (2.0, 0.3, 1.1, 1.9, 0.8)])
def test_eq8_pdf_integrates_to_product(alphas):
    def pdf(x):
        Fs = [x ** al for al in alphas]
        fs = [al * x ** (al - 1) for al in alphas]
        return oracle.eq8_pdf(Fs, fs)
    for x in (0.2, 0.5, 0.9, 1.0):
        val, err = quad(pdf, 0.0, x, limit=200)
        assert val == pytest.approx(x ** sum(alphas), abs=1e-7)


@pytest.mark.parametrize("seed", range(5))
def test_eq8_cdf_exact_rationals(seed):
    rng = np.random.default_rng(seed)
    k = int(rng.integers(1, 7))
    Fs = [Fraction(int(rng.integers(0, 17)), 16) for _ in range(k)]
    prod = Fraction(1)
    for f in Fs:
        prod *= f
    assert oracle.eq8_cdf(Fs) == prod


def test_eq8_iid_reduces_to_eq6():
    F, f = Fraction(3, 7), Fraction(2, 5)
    for k in range(1, 7):
        assert oracle.eq8_pdf([F] * k, [f] * k) == k * F ** (k - 1) * f


@pytest.mark.parametrize("seed", range(4))
def test_oracle_G_equals_integrated_eq8(seed):
    rng = np.random.default_rng(100 + seed)
    D, B, k = 5, 9, int(rng.integers(2, 7))
    counts = rng.integers(0, 6, (D, B)).astype(np.uint32)
    counts[:, -1] += 1
    F = oracle.cdf(counts)
    dist = rng.integers(0, D, k).astype(np.int32)
    a = np.zeros(k, np.int64)
    w = np.ones(k, np.int64)
    tot = counts.astype(np.int64).sum(1)
    cum = np.cumsum(counts.astype(np.int64), axis=1)
    for i in range(1, B + 1):
        r = oracle.score(F, a, w, [0, k], np.full(k, i), dist, [0], want_P=True)
        G = r["P"][0][k * (k - 1) // 2]
        Fs = [Fraction(int(cum[d, i - 1]), int(tot[d])) for d in dist]
        assert G == pytest.approx(float(oracle.eq8_cdf(Fs)), abs=1e-14)
