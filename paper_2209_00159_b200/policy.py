"""Replay policy thresholds: marshalling for the exact host-side computations
in liborloj (include/orloj.h, csrc/thresholds.cu).

A request of distribution d is dropped at time t iff D_r - t < thr[d]
(`orloj_replay_trace_ex`).  Rules:

* hopeless (A16): P_r(1) = 0 exactly  <=>  D_r - t < a_1 + w_1 m_min(d), with
  m_min(d) the first non-empty bin -- what the kernel uses when no thresholds
  are given (`hopeless_thresholds` only spells it out for tests: an index);
* expected latency (Alg. 1's drop, EstimateBatchLatency(r, 1)
  under the E_k scorer's model): orloj_expected_latency_thresholds;
* Alg. 1 per-batch-size feasibility, D_r - t >= ceil(E[L_bs]) of the
  all-application batch model: orloj_alg1_size_thresholds.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _abi


def _profile(offset_ticks, ticks_per_bin):
    a = np.ascontiguousarray(offset_ticks, dtype=np.int64)
    w = np.ascontiguousarray(ticks_per_bin, dtype=np.int64)
    if a.shape != w.shape or a.ndim != 1:
        raise _abi.OrlojError(1, "offset_ticks / ticks_per_bin must be 1-D of equal length")
    return a, w, _abi.LatencyProfile(len(a), a.ctypes.data, w.ctypes.data)


def _counts(counts):
    c = np.ascontiguousarray(counts, dtype=np.uint32)
    if c.ndim != 2:
        raise _abi.OrlojError(1, "counts must be [D, B]")
    return c


def expected_latency_thresholds(counts, offset_ticks, ticks_per_bin) -> np.ndarray:
    c = _counts(counts)
    a, w, prof = _profile(offset_ticks, ticks_per_bin)
    out = np.empty(c.shape[0], np.int64)
    _abi.check(_abi.lib().orloj_expected_latency_thresholds(c.ctypes.data, c.shape[0], c.shape[1],
                                                            ctypes.byref(prof), out.ctypes.data))
    return out


def hopeless_thresholds(counts, offset_ticks, ticks_per_bin) -> np.ndarray:
    counts = np.asarray(counts)
    m_min = np.argmax(counts > 0, axis=1) + 1
    return (int(offset_ticks[0]) + int(ticks_per_bin[0]) * m_min).astype(np.int64)


def alg1_size_thresholds(counts, offset_ticks, ticks_per_bin, weights=None) -> np.ndarray:
    c = _counts(counts)
    a, w, prof = _profile(offset_ticks, ticks_per_bin)
    wt = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    out = np.empty(len(a), np.int64)
    _abi.check(_abi.lib().orloj_alg1_size_thresholds(c.ctypes.data, c.shape[0], c.shape[1],
                                                     None if wt is None else wt.ctypes.data, ctypes.byref(prof),
                                                     out.ctypes.data))
    return out
