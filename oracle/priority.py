"""ORACLE — test infrastructure only (never on the product path).

Plain fp64 numpy implementation of the Eq. 1-2 priority score of a request
under batching (PAPER.md:423-455 Eq. 1-2, :571-593 batch latency / batch
formation) and of PopBatch (Alg. 1): SURVEY §8(f) item 2.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` may import it;
it shares no code with ``paper_2209_00159_b200``.

Readings (R10-R12):
  * L of a request is the latency of its whole batch.  For batch
    size bs the batch is bs i.i.d. draws from the mixture of all application
    distributions of the model, so F_L = F_mix^bs (Eq. 6), with
    the A1 grid: bin i of L_bs is (l1, l2] = (a + w(i-1), a + w i].
  * Eq. 2 treats each histogram bin as a uniform density h = pm_i / w over
    its range (the paper's "frequency h" must be a density for Eq. 2 to be
    E[C_delay] - E[C_now]; the pins below check exactly that).
  * Cost c = 1 for every request (one SLO class); E[L] is the mean
    of the same histogram, sum_i pm_i (l1 + l2) / 2.
"""
from __future__ import annotations

import numpy as np


def mixture_cdf(counts, weights=None, store_fp32=False) -> np.ndarray:
    """F_mix(tau_i) for i = 1..B: the weighted mixture of the applications'
    histogram CDFs ("all execution time distributions associated
    with the model").  counts [D][B] (every row with a positive total).
    store_fp32: read each F_d through the store's data format (log2 F rounded
    to fp32, include/orloj.h orloj_store) instead of exactly."""
    c = np.asarray(counts, dtype=np.float64)
    F = np.cumsum(c, axis=1) / c.sum(axis=1, keepdims=True)
    if store_fp32:
        with np.errstate(divide="ignore"):
            F = np.exp2(np.log2(F).astype(np.float32).astype(np.float64))
    wts = np.ones(c.shape[0]) if weights is None else np.asarray(weights, dtype=np.float64)
    return (wts[:, None] * F).sum(axis=0) / wts.sum()


def batch_latency_logpmf(counts, bs, weights=None, store_fp32=False) -> np.ndarray:
    """log pm_i, pm_i = P(L_bs in bin i), i = 1..B: the max of bs i.i.d. mixture
    draws (Eq. 6 with identical factors), G = F_mix^bs differenced.  Evaluated
    as log G_i = bs log F_mix and log(G_i - G_{i-1}) = log G_i +
    log(1 - exp(log G_{i-1} - log G_i)), the same quantity without the fp64
    underflow of F^bs for small F and large bs."""
    F = mixture_cdf(counts, weights, store_fp32)
    F[-1] = 1.0
    with np.errstate(divide="ignore"):
        lG = bs * np.log(F)
    prev = np.concatenate([[-np.inf], lG[:-1]])
    out = np.full(lG.shape, -np.inf)
    pos = lG > prev
    out[pos] = lG[pos] + np.log(-np.expm1(prev[pos] - lG[pos]))
    return out


def batch_latency_pmf(counts, bs, weights=None, store_fp32=False) -> np.ndarray:
    """pm_i = P(L_bs in bin i), i = 1..B (linear; see batch_latency_logpmf)."""
    return np.exp(batch_latency_logpmf(counts, bs, weights, store_fp32))


def expected_latency(pm, a, w) -> float:
    """E[L] of the histogram with uniform bins (l1, l2]: sum pm_i (l1 + l2)/2."""
    i = np.arange(1, len(pm) + 1, dtype=np.float64)
    return float(np.sum(pm * (a + w * (i - 0.5))))


def log_priority(pm, a, w, b, sigma) -> np.ndarray:
    """log p from the bin masses pm (see log_priority_lp)."""
    with np.errstate(divide="ignore"):
        return log_priority_lp(np.log(np.asarray(pm, dtype=np.float64)), a, w, b, sigma)


def log_priority_lp(lpm, a, w, b, sigma) -> np.ndarray:
    """log p for slacks sigma = D - t (array), Eq. 2 bin by bin:
         t <  D - l2:        (h/(E[L] b)) (e^{b l2} - e^{b l1}) e^{-b D} e^{b t}
         D - l2 <= t < D - l1: h/(E[L] b) - (h/(E[L] b)) e^{b l1} e^{-b D} e^{b t}
         D - l1 <= t:        0
       with c = 1 and h = pm_i / w, combined p = sum_i p_i.  Each term is
       evaluated as its logarithm (e^{b l2} e^{-bD} e^{bt} = e^{-b(sigma - l2)})
       and the sum by logaddexp, so no term overflows."""
    lpm = np.asarray(lpm, dtype=np.float64)
    sig = np.atleast_1d(np.asarray(sigma, dtype=np.float64))
    EL = expected_latency(np.exp(lpm), a, w)
    out = np.full(sig.shape, -np.inf)
    for i in range(1, len(lpm) + 1):
        if lpm[i - 1] == -np.inf:
            continue
        l1, l2 = a + w * (i - 1), a + w * i
        logh_b = lpm[i - 1] - np.log(w * b)  # log(h / b), h = pm_i / w
        term = np.full(sig.shape, -np.inf)
        full = sig >= l2
        part = (sig > l1) & (sig < l2)
        # (e^{b l2} - e^{b l1}) e^{-b sigma} = e^{-b (sigma - l2)} (1 - e^{-b w})
        term[full] = logh_b - b * (sig[full] - l2) + np.log1p(-np.exp(-b * w))
        # 1 - e^{b l1} e^{-b sigma} = 1 - e^{-b (sigma - l1)}
        term[part] = logh_b + np.log1p(-np.exp(-b * (sig[part] - l1)))
        out = np.logaddexp(out, term)
    return out - np.log(EL)


def scores(counts, a, w, num_sizes, b, offsets, deadline, now, weights=None, store_fp32=False) -> np.ndarray:
    """log p [N][num_sizes] for queue members (offsets relative to offsets[0]),
    slack D_r - now[q]; a, w are the profile arrays (index bs-1)."""
    off = np.asarray(offsets, dtype=np.int64) - int(offsets[0])
    dl = np.asarray(deadline, dtype=np.int64)
    out = np.empty((int(off[-1]), num_sizes))
    sig = np.empty(int(off[-1]), dtype=np.int64)
    for q in range(len(off) - 1):
        sig[off[q]:off[q + 1]] = dl[off[q]:off[q + 1]] - int(now[q])
    for bs in range(1, num_sizes + 1):
        lpm = batch_latency_logpmf(counts, bs, weights, store_fp32)
        out[:, bs - 1] = log_priority_lp(lpm, float(a[bs - 1]), float(w[bs - 1]), b, sig)
    return out


def log_priority_steps(pm, a, w, b, sigma, offsets, costs) -> np.ndarray:
    with np.errstate(divide="ignore"):
        return log_priority_steps_lp(np.log(np.asarray(pm, dtype=np.float64)), a, w, b, sigma, offsets, costs)


def log_priority_steps_lp(lpm, a, w, b, sigma, offsets, costs) -> np.ndarray:
    """Piecewise-step cost (Appendix): deadlines D + offsets[s]
    with cumulative costs costs[s] decompose into single steps (deadline
    D + offsets[s], cost costs[s] - costs[s-1]); the priority is the sum of
    the single-step priorities (each Eq. 2 with c = that increment)."""
    sig = np.atleast_1d(np.asarray(sigma, dtype=np.float64))
    out = np.full(sig.shape, -np.inf)
    prev = 0.0
    for off, c in zip(offsets, costs):
        out = np.logaddexp(out, np.log(c - prev) + log_priority_lp(lpm, a, w, b, sig + off))
        prev = c
    return out


def scores_steps(counts, a, w, num_sizes, b, offsets, deadline, now, step_offsets, step_costs, weights=None,
                 store_fp32=False) -> np.ndarray:
    """log p [N][num_sizes] under a piecewise-step cost (see log_priority_steps)."""
    off = np.asarray(offsets, dtype=np.int64) - int(offsets[0])
    dl = np.asarray(deadline, dtype=np.int64)
    out = np.empty((int(off[-1]), num_sizes))
    sig = np.empty(int(off[-1]), dtype=np.int64)
    for q in range(len(off) - 1):
        sig[off[q]:off[q + 1]] = dl[off[q]:off[q + 1]] - int(now[q])
    for bs in range(1, num_sizes + 1):
        lpm = batch_latency_logpmf(counts, bs, weights, store_fp32)
        out[:, bs - 1] = log_priority_steps_lp(lpm, float(a[bs - 1]), float(w[bs - 1]), b, sig, step_offsets,
                                               step_costs)
    return out


def store_rounding_eta(counts) -> np.ndarray:
    """eta_i >= |F^_d(tau_i) / F_d(tau_i) - 1| for every application d, where
    F^ = 2^{fl32(log2 F)} is F read through the store format (one RN rounding
    of log2 F to fp32: |dx| <= 2^-24 |x|, plus 2^-20 of that for a last-place
    error of the fp64 log2 before it): eta = e^{ln 2 * 2^-24 (1 + 2^-20) |log2 F|} - 1.
    F = 0 and F = 1 are exact (-inf and 0.0f), so they contribute 0; bin B is
    forced to 1 on both sides."""
    c = np.asarray(counts, dtype=np.float64)
    F = np.cumsum(c, axis=1) / c.sum(axis=1, keepdims=True)
    with np.errstate(divide="ignore"):
        x = np.abs(np.log2(F))
    x[~np.isfinite(x)] = 0.0
    eta = np.expm1(np.log(2.0) * 2.0 ** -24 * (1 + 2.0 ** -20) * x).max(axis=0)
    eta[-1] = 0.0
    return eta


def store_rounding_log_priority_bound(counts, a, w, b, sigma, bs, weights=None) -> np.ndarray:
    """First-order bound on |log p(F^) - log p(F)| for one batch size: how far
    the store format alone (log2 F rounded once to fp32) can move the Eq. 2
    priority of the exact histogram model.  The mixture CDF moves by at most
    eta_i relatively (a weighted mean of per-application factors), G_i = F^bs
    by gamma_i = G_i ((1 + eta_i)^bs - 1), a bin mass pm_i = G_i - G_{i-1} by
    dpm_i = gamma_i + gamma_{i-1}.  With T_i(sigma) >= 0 the per-unit-mass
    Eq. 2 term of bin i, p E[L] = sum pm_i T_i moves by at most
    r = sum dpm_i T_i / sum pm_i T_i relatively and E[L] = sum pm_i mid_i by
    r_L = sum dpm_i mid_i / E[L]; |d log p| <= r/(1-r) + r_L/(1-r_L)
    (|log(1+d)| <= |d|/(1-|d|)).  inf where r >= 1 (bins whose mass the
    rounding may erase decide p: near-empty bins at large bs)."""
    F = mixture_cdf(counts, weights)
    F[-1] = 1.0
    eta = store_rounding_eta(counts)
    G = F ** bs
    gam = G * np.expm1(bs * np.log1p(eta))
    dpm = gam + np.concatenate([[0.0], gam[:-1]])
    lpm = batch_latency_logpmf(counts, bs, weights)
    pm = np.exp(lpm)
    sig = np.atleast_1d(np.asarray(sigma, dtype=np.float64))
    B = len(pm)
    i = np.arange(1, B + 1, dtype=np.float64)
    EL = float(np.sum(pm * (a + w * (i - 0.5))))
    rL = float(np.sum(dpm * (a + w * (i - 0.5)))) / EL
    lnum = np.full(sig.shape, -np.inf)      # log sum dpm_k T_k, log domain (e^{-b sigma} underflows)
    lden = np.full(sig.shape, -np.inf)      # log sum pm_k T_k
    with np.errstate(divide="ignore"):
        ldpm = np.log(dpm)
    for k in range(1, B + 1):
        l1, l2 = a + w * (k - 1), a + w * k
        lT = np.full(sig.shape, -np.inf)
        full = sig >= l2
        part = (sig > l1) & (sig < l2)
        lT[full] = -b * (sig[full] - l2) + np.log(-np.expm1(-b * w)) - np.log(w * b)
        lT[part] = np.log(-np.expm1(-b * (sig[part] - l1))) - np.log(w * b)
        lnum = np.logaddexp(lnum, ldpm[k - 1] + lT)
        lden = np.logaddexp(lden, lpm[k - 1] + lT)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(np.isfinite(lden), np.exp(lnum - lden), np.inf)
        out = r / (1.0 - r) + rL / (1.0 - rL)
    out[~(r < 1.0)] = np.inf
    return out


def pop_batch(logp_rows, bs, num_sizes, cap=256) -> list[int]:
    """PopBatch (Alg. 1 line 18): the (up to) bs members with the highest
    priority for size bs, highest first, ties to the earlier member, members
    with p = 0 (log p = -inf) or NaN never selected; only the first `cap`
    members are candidates (the ABI's window)."""
    if not (1 <= bs <= num_sizes):
        return []
    cand = [(-float(v), r) for r, v in enumerate(logp_rows[:cap, bs - 1])
            if not (np.isnan(v) or v == -np.inf)]
    return [r for _, r in sorted(cand)[:bs]]
