"""ORACLE — test infrastructure only (never on the product path).

Scoring-model variants, plain fp64 Python loops for
small cases: the expected finish count
    E_k = sum_{r<=k} sum_s dc_s P(t + L_{B_k} <= D_r + off_s)
with a duration table dur[k-1][m] (m = 0..B, the batch time when the slowest
member sits at bin position m; Eq. 3-4 give a_k + w_k m), the
bin model
    * "edge": every bin's mass at its upper edge (A1), the batch time of a
      max bin i being dur[k-1][i]:  P = prod_j F_j(i*), i* = #{m >= 1 : dur[m] <= x};
    * "uniform": each member's position uniform within its bin (linear CDF
      inside bins) and the batch time dur linear between grid
      positions:  P = prod_j F_j^lin(m + u) for dur[m] <= x < dur[m+1];
and a piecewise-step cost (Appendix) with cumulative costs c_s
(dc_s = c_s - c_{s-1}).  Only ``tests/`` may import it; no code is shared
with ``paper_2209_00159_b200``.
"""
from __future__ import annotations

import numpy as np


def cdf_rows(counts) -> np.ndarray:
    """F_d(tau_i), i = 1..B, from integer counts."""
    c = np.asarray(counts, dtype=np.float64)
    return np.cumsum(c, axis=1) / c.sum(axis=1, keepdims=True)


def finish_prob(F, dists, dur_k, x, interpolate: bool) -> float:
    """P(batch of the members `dists` finishes within x ticks)."""
    B = F.shape[1]
    if not interpolate:
        i = int(np.sum(dur_k[1:] <= x))
        if i == 0:
            return 0.0
        p = 1.0
        for d in dists:
            p *= F[d, i - 1]
        return p
    if x < dur_k[0]:
        return 0.0
    m = int(np.nonzero(dur_k <= x)[0][-1])  # largest grid position with dur <= x
    if m == B:
        return 1.0
    u = (x - dur_k[m]) / (dur_k[m + 1] - dur_k[m])
    p = 1.0
    for d in dists:
        f0 = 0.0 if m == 0 else F[d, m - 1]
        f1 = F[d, m]
        p *= f0 + u * (f1 - f0)
    return p


def score(counts, dur, offsets, deadline, dist, now, interpolate=False, step_offsets=(0,), step_costs=(1.0,)):
    """E [Q][kmax] (zeros beyond K) and best_k [Q] (ties -> smallest k)."""
    F = cdf_rows(counts)
    dur = np.asarray(dur, dtype=np.int64)
    kmax = dur.shape[0]
    dc = np.diff(np.concatenate([[0.0], np.asarray(step_costs, dtype=np.float64)]))
    off = np.asarray(offsets, dtype=np.int64) - int(offsets[0])
    Q = len(off) - 1
    E = np.zeros((Q, kmax))
    best = np.zeros(Q, np.int32)
    for q in range(Q):
        n = int(off[q + 1] - off[q])
        K = min(n, kmax)
        sig = [int(deadline[off[q] + r]) - int(now[q]) for r in range(K)]
        ds = [int(dist[off[q] + r]) for r in range(K)]
        for k in range(1, K + 1):
            e = 0.0
            for r in range(k):
                for o, c in zip(step_offsets, dc):
                    e += c * finish_prob(F, ds[:k], dur[k - 1], sig[r] + int(o), interpolate)
            E[q, k - 1] = e
        if K:
            best[q] = int(np.argmax(E[q, :K])) + 1
    return E, best
