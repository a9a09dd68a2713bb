"""ORACLE — test infrastructure only (never on the product path).

Trace replay under the paper's scheduler iteration, Alg. 1,
for small traces (plain Python loops): SURVEY §8(f) item 1, the
"paper-faithful Alg. 1 policy in the replay driver".  Only ``tests/`` may
import it; it shares no code with ``paper_2209_00159_b200``.

Per scenario the replay state is the same as O2 (oracle.c, readings A9, A11,
A15-A17): constant SLO, so deadline order = arrival order; the window holds
the kmax earliest-deadline pending requests.  Each decision at time t:
  * drop (Alg. 1 l.10-13): r is removed from Q_bs iff t + E[L_bs] > D_r; it is
    timed out once infeasible for every bs, i.e. for bs = 1 (E[L_bs] grows
    with bs) -- applied when the window is scanned, like O2's drop;
  * Q_bs = {r : D_r - t >= thr_bs}, thr_bs = ceil(E[L_bs]) (integer ticks);
  * candidate (l.14-19): among bs with |Q_bs| >= bs, the earliest D_{Q_bs},
    ties -> larger bs (reading R14: the prose "overall earliest deadline");
  * PopBatch (l.20): the bs members of Q_bs with the highest Eq. 1-2 priority
    (oracle.priority, fp64), ties -> earlier member;
  * dispatch as O2 (duration a_bs + w_bs max true bin; finished iff
    t + dur <= D_r); the unpopped members stay pending, in order.
E[L_bs] is the all-application batch model: bs i.i.d. draws from
the weighted mixture, each bin uniform (Eq. 2's histogram), computed here in
exact rationals.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

from . import priority as pr


def size_thresholds(counts, a, w, weights=None) -> np.ndarray:
    """thr_bs = ceil(E[L_bs]), bs = 1..len(a), in exact rational arithmetic:
    E[L_bs] = a_bs + w_bs sum_i (F_mix(tau_i)^bs - F_mix(tau_{i-1})^bs) (i - 1/2)."""
    counts = np.asarray(counts)
    D, B = counts.shape
    wts = [Fraction(1)] * D if weights is None else [Fraction(float(x)) for x in weights]
    tot = [sum(int(c) for c in row) for row in counts]
    F = []
    for i in range(B):
        f = sum((wts[d] * Fraction(sum(int(c) for c in counts[d, :i + 1]), tot[d]) for d in range(D)), Fraction(0))
        F.append(f / sum(wts))
    F[-1] = Fraction(1)
    out = np.empty(len(a), np.int64)
    for k in range(len(a)):
        e = Fraction(int(a[k]))
        prev = Fraction(0)
        for i, f in enumerate(F):
            g = f ** (k + 1)
            e += int(w[k]) * (g - prev) * Fraction(2 * i + 1, 2)
            prev = g
        out[k] = math.ceil(e)
    return out


def replay(counts, a, w, b, arr_off, arrival, dist, true_bin, slo, thr, weights=None, follow_log=None,
           want_log=False):
    """Alg. 1 replay.  Returns dict(counters [S,7], log | None, ties [S,3]) with
    the same layout as oracle.replay; in follow mode (follow_log = the GPU's
    popped-member masks) the GPU's choice is applied when it is in the tie set
    (same candidate size, popped members inside Q_bs, and no unpopped member of
    Q_bs with a priority above a popped one by more than the fp32 tolerance of
    the priorities); ties[:, 2] is the first decision outside it."""
    kmax = len(a)
    S = len(slo)
    N = int(arr_off[-1]) if S else 0
    lpm = [pr.batch_latency_logpmf(counts, k + 1, weights, store_fp32=True) for k in range(kmax)]
    counters = np.zeros((S, 7), np.int64)
    log = np.zeros(N + S, np.int32) if want_log else None
    ties = np.zeros((S, 3), np.int64)
    for s in range(S):
        base, n = int(arr_off[s]), int(arr_off[s + 1] - arr_off[s])
        arr = [int(x) for x in arrival[base:base + n]]
        tb = [int(x) for x in true_bin[base:base + n]]
        sl = int(slo[s])
        t = -(1 << 63)
        cursor, carry = 0, []
        c_fin = c_drop = c_late = c_bat = c_busy = 0
        ndec, nties, first_bad = 0, 0, -1
        while cursor < n or carry:
            if not carry and arr[cursor] > t:
                t = arr[cursor]
            win = []
            for r in carry:
                if arr[r] + sl - t < thr[0]:
                    c_drop += 1
                else:
                    win.append(r)
            while len(win) < kmax and cursor < n and arr[cursor] <= t:
                r = cursor
                cursor += 1
                if arr[r] + sl - t < thr[0]:
                    c_drop += 1
                else:
                    win.append(r)
            carry = []
            if not win:
                continue
            wc = len(win)
            sig = [arr[r] + sl - t for r in win]
            # Q_bs: first member with slack >= thr_bs; candidate: earliest D_{Q_bs}, ties -> larger bs
            best = None
            for bs in range(1, min(kmax, wc) + 1):
                first = next((j for j in range(wc) if sig[j] >= thr[bs - 1]), wc)
                if wc - first >= bs and (best is None or sig[first] <= best[1]):
                    best = (bs, sig[first], first)
            bs, _, first = best
            lp = pr.log_priority_lp(lpm[bs - 1], float(a[bs - 1]), float(w[bs - 1]), b,
                                    np.array(sig[first:], dtype=np.float64))
            order = sorted(range(first, wc), key=lambda j: (-lp[j - first], j))
            pop = sorted(order[:bs])
            mask_o = sum(1 << j for j in pop)
            if follow_log is not None:
                mg = int(np.uint32(follow_log[base + s + ndec]))
                sel = [j for j in range(32) if (mg >> j) & 1]
                fin_lp = [abs(x) for x in lp if np.isfinite(x)]
                tol = 2.0 * (1e-6 + 2.0 ** -22 * (max(fin_lp) if fin_lp else 0.0))
                ok = len(sel) == bs and all(first <= j < wc for j in sel)
                if ok:
                    lo_sel = min(lp[j - first] for j in sel)
                    hi_rest = max([lp[j - first] for j in range(first, wc) if j not in sel], default=-np.inf)
                    ok = hi_rest <= lo_sel + tol or (hi_rest == -np.inf)
                if not ok and first_bad < 0:
                    first_bad = ndec
                if mg != mask_o:
                    nties += 1
                if ok:
                    pop = sel
            if log is not None:
                log[base + s + ndec] = np.int32(np.uint32(sum(1 << j for j in pop)))
            ndec += 1
            m = max(tb[win[j]] for j in pop)
            dur = int(a[bs - 1]) + int(w[bs - 1]) * m
            for j in pop:
                if t + dur <= arr[win[j]] + sl:
                    c_fin += 1
                else:
                    c_late += 1
            c_bat += 1
            c_busy += dur
            t += dur
            ps = set(pop)
            carry = [win[j] for j in range(wc) if j not in ps]
        if log is not None:
            log[base + s + ndec] = 0
        counters[s] = (n, c_fin, c_drop, c_late, c_bat, c_busy, t - arr[0] if n else 0)
        ties[s] = (ndec, nties, first_bad)
    return {"counters": counters, "log": log, "ties": ties}
