"""Replay drop thresholds (host logic, exact integers).

A request of distribution d is dropped at time t iff D_r - t < thr[d]
(`orloj_replay_trace_ex`).  Two rules:

* hopeless (A16): P_r(1) = 0 exactly  <=>  D_r - t < a_1 + w_1 m_min(d), where
  m_min(d) is the first non-empty bin (this is what the kernel uses when no
  thresholds are given);
* expected latency (Alg. 1's drop, EstimateBatchLatency(r, 1) =
  a_1 + w_1 E[bin_d] by Eq. 3 / Eq. 5 for a batch of one):
  t + a_1 + w_1 E[bin_d] > D_r  <=>  D_r - t - a_1 < w_1 E[bin_d]
  <=>  D_r - t < a_1 + ceil(w_1 sum_i i c_i / sum_i c_i)   (D_r - t is an integer),
  computed here in exact integer arithmetic from the histogram counts.

Alg. 1 (objective "alg1") uses per-batch-size thresholds instead: r is viable
for bs iff t + E[L_bs] <= D_r, E[L_bs] of the all-application batch
model (bs i.i.d. draws from the weighted mixture, uniform within a
bin as in Eq. 2), i.e. D_r - t >= ceil(E[L_bs]) -- `alg1_size_thresholds`,
exact rationals.
"""
from __future__ import annotations

import numpy as np


def expected_latency_thresholds(counts, offset_ticks, ticks_per_bin) -> np.ndarray:
    counts = np.asarray(counts)
    a1, w1 = int(offset_ticks[0]), int(ticks_per_bin[0])
    out = np.empty(counts.shape[0], np.int64)
    bins = np.arange(1, counts.shape[1] + 1, dtype=object)
    for d, row in enumerate(counts.astype(object)):
        num = int((bins * row).sum())
        den = int(row.sum())
        if den == 0:
            raise ValueError("cold start: histogram with total 0")
        out[d] = a1 + (w1 * num + den - 1) // den
    return out


def hopeless_thresholds(counts, offset_ticks, ticks_per_bin) -> np.ndarray:
    counts = np.asarray(counts)
    a1, w1 = int(offset_ticks[0]), int(ticks_per_bin[0])
    m_min = np.argmax(counts > 0, axis=1) + 1
    return (a1 + w1 * m_min).astype(np.int64)


def alg1_size_thresholds(counts, offset_ticks, ticks_per_bin, weights=None) -> np.ndarray:
    """thr_bs = ceil(E[L_bs]) for bs = 1..kmax, exactly: F_mix(tau_i) = N_i / M
    over a common denominator, G_i = (N_i / M)^bs, and
    E[L_bs] = a_bs + w_bs sum_i (G_i - G_{i-1}) (i - 1/2)
            = a_bs + w_bs X / (2 M^bs),  X = sum_i (N_i^bs - N_{i-1}^bs)(2i - 1)."""
    from fractions import Fraction
    from math import lcm

    counts = np.asarray(counts)
    D, B = counts.shape
    wts = [Fraction(1)] * D if weights is None else [Fraction(float(x)) for x in weights]
    if any(x < 0 for x in wts) or sum(wts) == 0:
        raise ValueError("weights must be >= 0 and not all 0")
    tot = [int(r.sum()) for r in counts.astype(object)]
    if min(tot) == 0:
        raise ValueError("cold start: histogram with total 0")
    cum = np.cumsum(counts.astype(object), axis=1)
    F = [sum((wts[d] * Fraction(int(cum[d, i]), tot[d]) for d in range(D)), Fraction(0)) / sum(wts)
         for i in range(B)]
    F[-1] = Fraction(1)
    M = 1
    for f in F:
        M = lcm(M, f.denominator)
    N = [f.numerator * (M // f.denominator) for f in F]
    out = np.empty(len(offset_ticks), np.int64)
    for k in range(len(offset_ticks)):
        bs = k + 1
        Mb = M ** bs
        prev, X = 0, 0
        for i, n in enumerate(N):
            g = n ** bs
            X += (g - prev) * (2 * (i + 1) - 1)
            prev = g
        wk = int(ticks_per_bin[k])
        out[k] = int(offset_ticks[k]) + (wk * X + 2 * Mb - 1) // (2 * Mb)
    return out
