"""ORACLE — test infrastructure only (never on the product path).

Plain fp64 CPU implementation of the Orloj batch-scoring path (SURVEY.md
§8(c) O1-O3), used to prove the CUDA path right.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import it.  It shares no code with
``paper_2209_00159_b200`` (and imports nothing from it).

The arithmetic lives in ``oracle.c`` (plain C + OpenMP over independent
queues / scenarios); this module only marshals numpy arrays.  The Python
helpers at the bottom (``eq8_*``) are the literal Eq. 8 evaluators used as
pins.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from fractions import Fraction
from itertools import combinations

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(HERE, "liboracle.so")
_lib = None

OK, EINVAL, ECOLD = 0, 1, 2
COUNTER_FIELDS = ("total", "finished", "dropped", "late", "batches", "busy_ticks", "span_ticks")


def build():
    """Compile oracle.c (gcc, OpenMP).  Building the checker is not using it."""
    src = os.path.join(HERE, "oracle.c")
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, src, "-lm"])


def _load():
    global _lib
    if _lib is None:
        src = os.path.join(HERE, "oracle.c")
        if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
            build()
        lib = ctypes.CDLL(_LIB)
        P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        lib.oracle_cdf.argtypes = [P, i32, i32, P]
        lib.oracle_score.argtypes = [P, i32, i32, P, P, i32, i64, P, P, P, P, P, P, P, P, P, i32]
        lib.oracle_bruteforce.argtypes = [P, i32, i32, P, P, i32, P, P, i64, P, P, i32]
        lib.oracle_replay.argtypes = [P, i32, i32, P, P, i32, i64, P, P, P, P, P, P, P, P, P, i32, i32, i32, P, P,
                                      P, P]
        for f in (lib.oracle_cdf, lib.oracle_score, lib.oracle_bruteforce, lib.oracle_replay,
                  lib.oracle_max_threads):
            f.restype = ctypes.c_int32
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class OracleError(RuntimeError):
    pass


def cdf(counts) -> np.ndarray:
    """F[d][i-1] = F_d(tau_i) in fp64 (A1)."""
    counts = _c(counts, np.uint32)
    D, B = counts.shape
    F = np.empty((D, B), np.float64)
    st = _load().oracle_cdf(_p(counts), D, B, _p(F))
    if st == ECOLD:
        raise OracleError("cold start: histogram with total 0")
    if st:
        raise OracleError(f"oracle_cdf status {st}")
    return F


def score(F, a, w, offsets, deadline, dist, now, want_P=False, want_EL=False, nthreads=0):
    """O1 over all queues.  Returns dict(E [Q,kmax], P [Q,T] | None, EL | None,
    best_k [Q], best_E [Q])."""
    F = _c(F, np.float64)
    a, w = _c(a, np.int64), _c(w, np.int64)
    offsets, deadline, now = _c(offsets, np.int64), _c(deadline, np.int64), _c(now, np.int64)
    dist = _c(dist, np.int32)
    D, B = F.shape
    kmax = len(a)
    Q = len(now)
    E = np.empty((Q, kmax), np.float64)
    P = np.empty((Q, kmax * (kmax + 1) // 2), np.float64) if want_P else None
    EL = np.empty((Q, kmax), np.float64) if want_EL else None
    bk = np.empty(Q, np.int32)
    bE = np.empty(Q, np.float64)
    st = _load().oracle_score(_p(F), D, B, _p(a), _p(w), kmax, Q, _p(offsets), _p(deadline), _p(dist),
                              _p(now), _p(E), _p(P), _p(EL), _p(bk), _p(bE), nthreads)
    if st:
        raise OracleError(f"oracle_score status {st}")
    return {"E": E, "P": P, "EL": EL, "best_k": bk, "best_E": bE}


def bruteforce(counts, a, w, deadline, dist, now, nthreads=0):
    """O3 for one queue of K = len(deadline) <= 12 members: (P packed, E)."""
    counts = _c(counts, np.uint32)
    D, B = counts.shape
    deadline, dist = _c(deadline, np.int64), _c(dist, np.int32)
    K = len(deadline)
    a, w = _c(a, np.int64), _c(w, np.int64)
    P = np.zeros(K * (K + 1) // 2, np.float64)
    E = np.zeros(K, np.float64)
    st = _load().oracle_bruteforce(_p(counts), D, B, _p(a), _p(w), K, _p(deadline), _p(dist), int(now),
                                   _p(P), _p(E), nthreads)
    if st:
        raise OracleError(f"oracle_bruteforce status {st}")
    return P, E


def replay(F, a, w, arr_off, arrival, dist, true_bin, slo, follow_log=None, want_log=False, nthreads=0,
           objective="expected_finish", drop="hopeless", counts=None, t_start=None, want_outcome=False):
    """O2.  Returns dict(counters [S,7] int64, log | None, ties [S,3]:
    (decisions, GPU choices != oracle choice, first decision outside the tie
    set or -1), t_end [S], outcome [N] uint8 | None (1 finished, 2 late,
    3 dropped)).  objective: "expected_finish" (argmax E_k) or "finish_rate"
    (argmax E_k / E[L_{B_k}]); drop: "hopeless" (A16) or "expected_latency"
    (Alg. 1; needs `counts`).  t_start [S]: the worker is busy
    until then (a feedback epoch continuing the previous one; None = free)."""
    F = _c(F, np.float64)
    D, B = F.shape
    a, w = _c(a, np.int64), _c(w, np.int64)
    arr_off, arrival, slo = _c(arr_off, np.int64), _c(arrival, np.int64), _c(slo, np.int64)
    dist, true_bin = _c(dist, np.int32), _c(true_bin, np.int16)
    S = len(slo)
    N = int(arr_off[-1]) if S else 0
    counters = np.zeros((S, 7), np.int64)
    log = np.zeros(N + S, np.int32) if want_log else None
    ties = np.zeros((S, 3), np.int64)
    fl = _c(follow_log, np.int32) if follow_log is not None else None
    obj = {"expected_finish": 0, "finish_rate": 1}[objective]
    dm = {"hopeless": 0, "expected_latency": 1}[drop]
    cts = None if counts is None else _c(counts, np.uint32)
    ts = None if t_start is None else _c(t_start, np.int64)
    t_end = np.zeros(S, np.int64)
    oc = np.zeros(N, np.uint8) if want_outcome else None
    st = _load().oracle_replay(_p(F), D, B, _p(a), _p(w), len(a), S, _p(arr_off), _p(arrival), _p(dist),
                               _p(true_bin), _p(slo), _p(counters), _p(fl), _p(log), _p(ties), nthreads, obj, dm,
                               _p(cts), _p(ts), _p(t_end), _p(oc))
    if st:
        raise OracleError(f"oracle_replay status {st}")
    return {"counters": counters, "log": log, "ties": ties, "t_end": t_end, "outcome": oc}


def bucket_counters(counters, bucket, num_buckets):
    """Sum per-scenario counters into per-bucket rows (integer, exact)."""
    out = np.zeros((num_buckets, 7), np.int64)
    np.add.at(out, np.asarray(bucket), counters)
    return out


# ----------------------------------------------------------------------------
# Eq. 8 literal evaluators (pins)
# ----------------------------------------------------------------------------

def eq8_pdf(Fs, fs):
    """Eq. 8 exactly as printed: f_(k) = sum_{kappa=1..k} (-1)^{k-kappa} kappa^k/k!
    * sum_{|s|=kappa} k [F^s]^{k-1} f^s, with F^s, f^s the subset means of Eq. 7
    (PAPER.md:517-525).  Fs, fs: the k CDF and PDF values at one point (any
    numeric type, e.g. Fraction)."""
    k = len(Fs)
    exact = all(isinstance(x, (Fraction, int)) for x in list(Fs) + list(fs))
    tot = Fraction(0) if exact else 0.0
    for kappa in range(1, k + 1):
        coef = Fraction(kappa ** k, math.factorial(k)) if exact else kappa ** k / math.factorial(k)
        inner = Fraction(0) if exact else 0.0
        for s in combinations(range(k), kappa):
            Fsub = sum(Fs[i] for i in s) / kappa
            fsub = sum(fs[i] for i in s) / kappa
            inner += k * Fsub ** (k - 1) * fsub
        tot += (-1) ** (k - kappa) * coef * inner
    return tot


def eq8_cdf(Fs):
    """Eq. 8 integrated term by term: d/dl [F^s]^k = k [F^s]^{k-1} f^s, so the CDF
    of the max is sum_kappa (-1)^{k-kappa} kappa^k/k! sum_{|s|=kappa} [F^s]^k.
    With exact rationals this is the literal subset-sum form the paper prints,
    evaluated without using the product of CDFs."""
    k = len(Fs)
    tot = Fraction(0)
    for kappa in range(1, k + 1):
        inner = Fraction(0)
        for s in combinations(range(k), kappa):
            inner += (sum((Fraction(Fs[i]) for i in s), Fraction(0)) / kappa) ** k
        tot += (-1) ** (k - kappa) * Fraction(kappa ** k, math.factorial(k)) * inner
    return tot
