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
