"""ORACLE — test infrastructure only (never on the product path).

The long-term feedback loop written
out step by step, reading R15:

  for epoch e = 0 .. E-1:
    replay the arrivals [floor(e n / E), floor((e+1) n / E)) of every scenario
      with the current store (static during the epoch, A18), the worker busy
      until the end of the scenario's previous epoch       (oracle.replay, O2)
    "finished requests are sampled and sent to the profiler to evaluate
      individually": every completed request (finished or late)
      with a sample bit adds its solo time -- its hidden true bin -- to the
      window histogram of its application
    "picked up and accumulated by the scheduler periodically":
      every application whose window holds >= min_samples samples gets its
      CDF rebuilt from the window (oracle.cdf); the others keep their rows
    "resets its profiling memory every once in a while": after
      epochs W-1, 2W-1, ... the window is emptied

Only ``tests/`` may import it; it shares no code with ``paper_2209_00159_b200``.
"""
from __future__ import annotations

import numpy as np

import oracle


def epoch_bounds(n: int, e: int, E: int) -> tuple[int, int]:
    """Arrivals [floor(e n / E), floor((e+1) n / E)) of a scenario of n arrivals."""
    return (e * n) // E, ((e + 1) * n) // E


def epoch_index(arr_off, e: int, E: int):
    """Global arrival indices of epoch e of every scenario, and its CSR offsets."""
    off = np.asarray(arr_off, dtype=np.int64)
    parts, lens = [], []
    for s in range(len(off) - 1):
        n = int(off[s + 1] - off[s])
        b0, b1 = epoch_bounds(n, e, E)
        parts.append(np.arange(off[s] + b0, off[s] + b1, dtype=np.int64))
        lens.append(b1 - b0)
    idx = np.concatenate(parts) if parts else np.zeros(0, np.int64)
    return idx, np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)


def epoch_log_view(log_full, arr_off, e: int, E: int) -> np.ndarray:
    """Epoch e's decisions, from a log in the [N + S] layout of one epoch call
    (decision d of scenario s at arr_off[s] + s + floor(e n_s / E) + d, then a
    0), rearranged into oracle.replay's layout for the epoch's sub-trace."""
    off = np.asarray(arr_off, dtype=np.int64)
    out = []
    for s in range(len(off) - 1):
        n = int(off[s + 1] - off[s])
        b0, b1 = epoch_bounds(n, e, E)
        p0 = int(off[s]) + s + b0
        out.append(np.asarray(log_full[p0:p0 + (b1 - b0) + 1]))
    return np.concatenate(out).astype(np.int32) if out else np.zeros(0, np.int32)


def replay_feedback(counts0, a, w, arr_off, arrival, dist, true_bin, slo, num_epochs: int, window_epochs: int,
                    min_samples: int, sample_mask=None, follow_logs=None, objective="expected_finish",
                    drop="hopeless"):
    """The loop above.  counts0: the prior histograms the first store is built
    from.  follow_logs: per-epoch logs in the [N + S] layout (the GPU's), for
    follow mode.  Returns dict(counters [E][S][7], ties [E][S][3], outcome [N],
    window [D][B] (the window the last refresh used), F [D][B] (the final
    store), refreshed [E][D] (rows rebuilt after each epoch))."""
    counts0 = np.asarray(counts0)
    D, B = counts0.shape
    F = oracle.cdf(counts0)
    arrival, dist, true_bin = np.asarray(arrival), np.asarray(dist), np.asarray(true_bin)
    slo = np.asarray(slo, dtype=np.int64)
    S = len(slo)
    N = int(np.asarray(arr_off)[-1]) if S else 0
    mask = np.ones(N, bool) if sample_mask is None else np.asarray(sample_mask) != 0
    t = np.full(S, np.iinfo(np.int64).min, np.int64)
    window = np.zeros((D, B), np.int64)
    outcome = np.zeros(N, np.uint8)
    counters, ties, refreshed = [], [], []
    last_window = window.copy()
    for e in range(num_epochs):
        idx, sub_off = epoch_index(arr_off, e, num_epochs)
        fl = None if follow_logs is None else epoch_log_view(follow_logs[e], arr_off, e, num_epochs)
        r = oracle.replay(F, a, w, sub_off, arrival[idx], dist[idx], true_bin[idx], slo, follow_log=fl,
                          objective=objective, drop=drop, counts=counts0 if drop != "hopeless" else None,
                          t_start=t, want_outcome=True)
        t = r["t_end"]
        oc = r["outcome"]
        outcome[idx] = oc
        counters.append(r["counters"])
        ties.append(r["ties"])
        done = ((oc == 1) | (oc == 2)) & mask[idx]
        np.add.at(window, (dist[idx][done], true_bin[idx][done].astype(np.int64) - 1), 1)
        rows = window.sum(axis=1) >= max(1, int(min_samples))
        for d in np.nonzero(rows)[0]:
            F[d] = oracle.cdf(window[d:d + 1])[0]
        refreshed.append(rows.copy())
        last_window = window.copy()
        if (e + 1) % window_epochs == 0:
            window[:] = 0
    return {"counters": np.stack(counters) if counters else np.zeros((0, S, 7), np.int64),
            "ties": np.stack(ties) if ties else np.zeros((0, S, 3), np.int64),
            "outcome": outcome, "window": last_window, "F": F, "refreshed": np.stack(refreshed)}
