"""Seeded synthetic inputs shared by the CUDA path and the oracle.

This module produces DATA only: integer histogram counts, deadlines, latency
profiles (Eq. 3 presets), arrival traces.  It holds none of the method's
arithmetic (no CDF products, bin lookups, finish probabilities or argmax) —
those live separately in ``oracle/`` (fp64 CPU) and
``paper_2209_00159_b200/csrc`` (CUDA), which share no code.

Floating point is used only to *shape* distributions (normal / lognormal
mixtures), after which everything is converted once, on the host, into exact
integer counts with total 2^30 (largest remainder), so both sides see the same
rationals.  Bulk C3 rows and C5 traces are expanded from those integers by the
integer-only generators in ``gen_common.h`` (host build ``gen_host.c`` and
device build ``gen_dev.cu``, bit-identical by construction).

The recipes follow SURVEY.md §8(d) and are restated in DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np
from scipy.special import ndtr

HERE = os.path.dirname(os.path.abspath(__file__))
SEED_BASE = 20220901
TOTAL = 1 << 30          # every histogram has exactly 2^30 counts
T0 = 1 << 40             # absolute tick origin (1 tick = 1 us): large on purpose
SNAPSHOT_SLO_MULTS = (1.5, 2.0, 3.0, 4.0, 5.0)
BUCKET_SLO_MULTS = (1.5, 2.0, 2.5, 3.0, 3.5, 4.0, 4.5, 5.0)


# ----------------------------------------------------------------------------
# integer histograms
# ----------------------------------------------------------------------------

def largest_remainder(pmf, total: int = TOTAL) -> np.ndarray:
    """Round a non-negative pmf to integer counts summing exactly to ``total``
    (largest remainder, ties to the lower bin index)."""
    pmf = np.asarray(pmf, dtype=np.float64)
    pmf = np.clip(pmf, 0.0, None)
    pmf = pmf / pmf.sum()
    raw = pmf * total
    base = np.floor(raw).astype(np.int64)
    short = int(total - base.sum())
    if short > 0:
        rem = raw - base
        order = np.lexsort((np.arange(len(rem)), -rem))
        base[order[:short]] += 1
    assert base.sum() == total and (base >= 0).all()
    return base.astype(np.uint32)


def binned_from_cdf(cdf, B: int, delta: int) -> np.ndarray:
    """pmf over B bins 'discrete at upper edges': bin i (1..B) holds
    the mass of (tau_{i-1}, tau_i], tau_i = i*delta; the lower tail folds into
    bin 1 and the upper tail into bin B."""
    edges = np.arange(1, B, dtype=np.float64) * delta
    c = cdf(edges)
    return np.diff(np.concatenate([[0.0], c, [1.0]]))


@dataclass
class Family:
    """A set of per-application execution-time histograms on one grid."""
    name: str
    counts: np.ndarray       # uint32 [D][B], each row sums to 2^30
    bin_ticks: int           # Delta
    target_mean_ms: float = float("nan")
    target_p99_ms: float = float("nan")

    @property
    def D(self):
        return self.counts.shape[0]

    @property
    def B(self):
        return self.counts.shape[1]

    def pooled_pmf(self) -> np.ndarray:
        return self.counts.astype(np.float64).sum(0) / (TOTAL * self.D)

    def mean_ticks(self) -> float:
        tau = np.arange(1, self.B + 1) * self.bin_ticks
        return float((self.pooled_pmf() * tau).sum())

    def mean_bin(self) -> float:
        return float((self.pooled_pmf() * np.arange(1, self.B + 1)).sum())

    def p99_ticks(self) -> int:
        """A19: the smallest tau_i whose pooled CDF is >= 0.99 (integer ticks)."""
        cum = np.cumsum(self.counts.astype(np.int64).sum(0))
        i = int(np.searchsorted(cum, math.ceil(0.99 * TOTAL * self.D)))
        return (i + 1) * self.bin_ticks

    def cum(self) -> np.ndarray:
        return np.cumsum(self.counts.astype(np.uint64), axis=1).astype(np.uint32)


def _normal_mix_cdf(centers, widths, weights):
    def cdf(x):
        return sum(w * ndtr((x - c) / s) for c, s, w in zip(centers, widths, weights))
    return cdf


def _lognormal_cdf(median, shape):
    def cdf(x):
        return ndtr((np.log(np.maximum(x, 1e-300)) - math.log(median)) / shape)
    return cdf


def dirichlet_family(seed: int, D: int = 8, B: int = 16, delta: int = 1000) -> Family:
    """C1: D distinct Dirichlet(1) pmfs over B bins."""
    rng = np.random.default_rng(seed)
    counts = np.stack([largest_remainder(rng.dirichlet(np.ones(B))) for _ in range(D)])
    return Family("dirichlet", counts, delta)


def skipnet_family(seed: int, D: int = 8, B: int = 64, delta: int = 100) -> Family:
    """SkipNet-like early exits: 3-cluster mixture (2.2 / 3.4 / 5.2 ms), weights
    fitted to Table 1's mean 3.24 ms / P99 5.56 ms, Dirichlet
    jittered per application."""
    rng = np.random.default_rng(seed)
    centers = (2200.0, 3400.0, 5200.0)
    widths = (150.0, 150.0, 250.0)
    w0 = np.array([0.328, 0.542, 0.130])
    rows = [largest_remainder(binned_from_cdf(_normal_mix_cdf(centers, widths, rng.dirichlet(400 * w0)), B, delta))
            for _ in range(D)]
    return Family("skipnet", np.stack(rows), delta, 3.24, 5.56)


def rdi_family(seed: int, D: int = 8, B: int = 64, delta: int = 46000) -> Family:
    """RDI-Nets-like: 4 exits (0.35 / 0.6 / 1.4 / 2.65 s), weights fitted to
    mean 683 ms / P99 2668 ms."""
    rng = np.random.default_rng(seed)
    centers = (350e3, 600e3, 1400e3, 2650e3)
    widths = tuple(0.06 * c for c in centers)
    w0 = np.array([0.232, 0.626, 0.120, 0.022])
    rows = [largest_remainder(binned_from_cdf(_normal_mix_cdf(centers, widths, rng.dirichlet(800 * w0)), B, delta))
            for _ in range(D)]
    return Family("rdi", np.stack(rows), delta, 683.0, 2668.0)


def gpt_family(seed: int, D: int = 8, B: int = 64, delta: int = 3790) -> Family:
    """GPT-Cornell-like variable-length generation: per-app lognormals, median
    92 ms x exp(N(0, 0.13)), shape U[0.15, 0.23]; population mean 94.84 /
    P99 161.69 ms."""
    rng = np.random.default_rng(seed)
    rows = []
    for _ in range(D):
        med = 92e3 * math.exp(rng.normal(0.0, 0.13))
        rows.append(largest_remainder(binned_from_cdf(_lognormal_cdf(med, rng.uniform(0.15, 0.23)), B, delta)))
    return Family("gpt", np.stack(rows), delta, 94.84, 161.69)


def static_family(B: int = 64, delta: int = 250, bins=(32, 28)) -> Family:
    """Static CNN (Inception / ResNet-like): exact point masses."""
    counts = np.zeros((len(bins), B), np.uint32)
    for d, b in enumerate(bins):
        counts[d, b - 1] = TOTAL
    return Family("static", counts, delta)


def point_family(B: int = 32, delta: int = 500, bins=(16, 10), near: bool = False) -> Family:
    """C4: exact point masses at bins 16 and 10 of 32 (Delta = 500 us); the
    'near' variant puts 1e-3 of the mass in the next bin."""
    counts = np.zeros((len(bins), B), np.uint32)
    for d, b in enumerate(bins):
        if near:
            pmf = np.zeros(B)
            pmf[b - 1] = 1 - 1e-3
            pmf[b] = 1e-3
            counts[d] = largest_remainder(pmf)
        else:
            counts[d, b - 1] = TOTAL
    return Family("point-near" if near else "point", counts, delta)


def bart_templates(seed: int, T: int = 4096, B: int = 256) -> Family:
    """C3 templates: per-request lognormal with median 765.7 ms x exp(N(0, 0.113))
    and shape U[0.05, 0.15]; the population matches BART-CNN mean 774.66 /
    P99 1101.99 ms.  Delta = ceil(1.5 * P99 / 256) us."""
    delta = math.ceil(1.5 * 1101990 / B)
    rng = np.random.default_rng(seed)
    rows = []
    for _ in range(T):
        med = 765.7e3 * math.exp(rng.normal(0.0, 0.113))
        rows.append(largest_remainder(binned_from_cdf(_lognormal_cdf(med, rng.uniform(0.05, 0.15)), B, delta)))
    return Family("bart", np.stack(rows), delta, 774.66, 1101.99)


# ----------------------------------------------------------------------------
# latency profiles (Eq. 3 presets)
# ----------------------------------------------------------------------------

@dataclass
class Profile:
    a: np.ndarray   # int64 [kmax], a_k (ticks)
    w: np.ndarray   # int64 [kmax], w_k (ticks per bin)

    @property
    def kmax(self):
        return len(self.a)


def eq3_profile(c0_ticks: float, c1: float, bin_ticks: int, kmax: int) -> Profile:
    """Eq. 3 on the bin grid: a_k = round(c0), w_k = round(c1*k*Delta)."""
    k = np.arange(1, kmax + 1)
    a = np.full(kmax, int(round(c0_ticks)), np.int64)
    w = np.array([int(round(c1 * kk * bin_ticks)) for kk in k], np.int64)
    return Profile(a, w)


def eq3_half(fam: Family, kmax: int) -> Profile:
    """'Eq3-half': c0 = 0.5 * mean, c1 = 0.5 (k = 1 ~ solo time on average)."""
    return eq3_profile(0.5 * fam.mean_ticks(), 0.5, fam.bin_ticks, kmax)


# ----------------------------------------------------------------------------
# queue snapshots (score / pick configs)
# ----------------------------------------------------------------------------

@dataclass
class Queues:
    offsets: np.ndarray    # int64 [Q+1]
    arrival: np.ndarray    # int64 [N]
    deadline: np.ndarray   # int64 [N]
    dist: np.ndarray       # int32 [N]
    now: np.ndarray        # int64 [Q]

    @property
    def Q(self):
        return len(self.now)

    @property
    def N(self):
        return int(self.offsets[-1])

    def subset(self, qs) -> "Queues":
        qs = np.asarray(qs, dtype=np.int64)
        lens = self.offsets[qs + 1] - self.offsets[qs]
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        idx = np.concatenate([np.arange(self.offsets[q], self.offsets[q + 1]) for q in qs]) if len(qs) else np.zeros(0, np.int64)
        idx = idx.astype(np.int64)
        return Queues(off, self.arrival[idx], self.deadline[idx], self.dist[idx], self.now[qs])


def snapshot_queues(seed: int, lengths, slo_base_ticks: int, dist_ids=None, D: int | None = None,
                    mults=SNAPSHOT_SLO_MULTS, now0: int = T0) -> Queues:
    """Queues are snapshots at t = now: SLO = m * P99 with m drawn
    per queue, request ages ~ U[0, SLO) sorted descending, so deadlines ascend;
    ties fall back to arrival then index order (A9)."""
    rng = np.random.default_rng(seed)
    lengths = np.asarray(lengths, np.int64)
    Q = len(lengths)
    off = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    N = int(off[-1])
    slo = np.round(np.asarray(mults)[rng.integers(0, len(mults), Q)] * slo_base_ticks).astype(np.int64)
    now = now0 + np.arange(Q, dtype=np.int64) * 1000
    u = rng.random(N)
    qid = np.repeat(np.arange(Q), lengths)
    ages = np.floor(u * slo[qid]).astype(np.int64)
    # sort ages descending within each queue
    if Q and (lengths == lengths[0]).all():
        ages = -np.sort(-ages.reshape(Q, -1), axis=1).reshape(-1)
    else:
        order = np.lexsort((-ages, qid))
        ages = ages[order]
    arrival = now[qid] - ages
    deadline = arrival + slo[qid]
    if dist_ids is None:
        dist_ids = rng.integers(0, D, N).astype(np.int32)
    return Queues(off, arrival.astype(np.int64), deadline.astype(np.int64), np.asarray(dist_ids, np.int32), now)


# ----------------------------------------------------------------------------
# configs C1..C4
# ----------------------------------------------------------------------------

@dataclass
class ScoreConfig:
    name: str
    fam: Family                # counts on host (for C3: the templates)
    profile: Profile
    queues: Queues
    rows: str = "family"       # "family": dist_id indexes fam.counts; "c3": dist_id indexes expanded rows
    n_rows: int = 0            # C3: number of expanded rows
    row_seed: int = 0

    @property
    def kmax(self):
        return self.profile.kmax


def config1() -> ScoreConfig:
    seed = SEED_BASE + 1
    fam = dirichlet_family(seed, D=8, B=16, delta=1000)
    prof = Profile(np.full(8, 1000, np.int64), 500 * np.arange(1, 9, dtype=np.int64))
    rng = np.random.default_rng(seed)
    sig = np.sort(rng.integers(5000, 60001, 8)).astype(np.int64)      # deadlines U[5, 60] ms
    now = np.array([T0], np.int64)
    dl = now[0] + sig
    q = Queues(np.array([0, 8], np.int64), np.full(8, now[0], np.int64), dl, rng.permutation(8).astype(np.int32), now)
    return ScoreConfig("C1", fam, prof, q)


def config2(Q: int = 1024, n: int = 64, kmax: int = 32) -> ScoreConfig:
    seed = SEED_BASE + 2
    fam = skipnet_family(seed)
    prof = eq3_half(fam, kmax)
    q = snapshot_queues(seed, np.full(Q, n), fam.p99_ticks(), D=fam.D)
    return ScoreConfig("C2", fam, prof, q)


def config_priority(Q: int = 65536, n: int = 256, sizes: int = 32) -> ScoreConfig:
    """P1: Eq. 1-2 priorities of every queued request for
    batch sizes 1..32 over the SkipNet-like application mix (8 apps, B 64), the
    C3 queue shape (65,536 queues x 256 requests)."""
    seed = SEED_BASE + 6
    fam = skipnet_family(seed)
    prof = eq3_half(fam, sizes)
    q = snapshot_queues(seed, np.full(Q, n), fam.p99_ticks(), D=fam.D)
    return ScoreConfig("P1", fam, prof, q)


def config3(Q: int = 65536, n: int = 256, kmax: int = 256, T: int = 4096, instance: int = 0) -> ScoreConfig:
    """Per-request rows: row ids are a seeded random permutation of [0, Q*n), so
    every candidate is a true 1 KB gather.  `instance` selects an
    independent draw of rows and queues (one per rank under weak scaling)."""
    seed = SEED_BASE + 3
    fam = bart_templates(seed, T=T)
    prof = eq3_half(fam, kmax)
    rng = np.random.default_rng(seed + 1000 + 7919 * instance)
    n_rows = Q * n
    perm = rng.permutation(n_rows).astype(np.int32)
    q = snapshot_queues(seed + 7919 * instance, np.full(Q, n), fam.p99_ticks(), dist_ids=perm)
    return ScoreConfig("C3", fam, prof, q, rows="c3", n_rows=n_rows, row_seed=seed + 7919 * instance)


def config4(Q: int = 1 << 20, n: int = 32, kmax: int = 32, near: bool = False) -> ScoreConfig:
    seed = SEED_BASE + 4
    fam = point_family(near=near)
    prof = eq3_half(fam, kmax)
    q = snapshot_queues(seed, np.full(Q, n), fam.p99_ticks(), D=fam.D)
    return ScoreConfig("C4-near" if near else "C4", fam, prof, q)


# ----------------------------------------------------------------------------
# C5 replay traces
# ----------------------------------------------------------------------------

C5_FAMILIES = ("skipnet", "rdi", "gpt", "static")
C5_SEEDS_PER_BUCKET = 256
C5_ARRIVALS = 100_000
C5_KMAX = 32
RHO1 = 0.9   # offered load if nothing were batched


def c5_family(name: str) -> Family:
    seed = SEED_BASE + 5
    return {"skipnet": lambda: skipnet_family(seed),
            "rdi": lambda: rdi_family(seed + 1),
            "gpt": lambda: gpt_family(seed + 2),
            "static": lambda: static_family()}[name]()


def exp_table_q16() -> np.ndarray:
    u = (np.arange(65536, dtype=np.float64) + 0.5) / 65536.0
    return np.round(-np.log(u) * 65536.0).astype(np.uint32)


@dataclass
class TraceFamily:
    """Everything needed to generate the C5 traces of one family."""
    fam: Family
    profile: Profile
    base_gap: int                 # mean inter-arrival ticks = E[dur(1)] / rho1
    exp_q16: np.ndarray
    cum: np.ndarray               # uint32 [D][B]
    seed: int
    findex: int

    def slo_of_bucket(self, b: int) -> int:
        m2 = int(round(2 * BUCKET_SLO_MULTS[b]))      # exact: 2*mult is an integer
        return (self.fam.p99_ticks() * m2) // 2


def c5_trace_family(name: str, kmax: int = C5_KMAX) -> TraceFamily:
    fam = c5_family(name)
    prof = eq3_half(fam, kmax)
    edur1 = prof.a[0] + prof.w[0] * fam.mean_bin()
    return TraceFamily(fam, prof, int(round(edur1 / RHO1)), exp_table_q16(), fam.cum(),
                       SEED_BASE + 5, C5_FAMILIES.index(name))


def c5_scenarios(tf: TraceFamily, seeds_per_bucket: int = C5_SEEDS_PER_BUCKET):
    """Local scenario u of a family: bucket = u % 8, seed index = u // 8.
    Global id (hashed) = findex * 2^20 + u.  Returns (global ids, bucket, slo)."""
    nb = len(BUCKET_SLO_MULTS)
    u = np.arange(nb * seeds_per_bucket, dtype=np.int64)
    bucket = (u % nb).astype(np.int32)
    gid = (tf.findex << 20) + u
    slo = np.array([tf.slo_of_bucket(b) for b in range(nb)], np.int64)[bucket]
    return gid.astype(np.uint64), bucket, slo


# ----------------------------------------------------------------------------
# native integer generators (host build + device build)
# ----------------------------------------------------------------------------

_host = None
_dev = None


def _host_lib():
    global _host
    if _host is None:
        path = os.path.join(HERE, "libgen_host.so")
        if not os.path.exists(path):
            build_host()
        _host = ctypes.CDLL(path)
        P = ctypes.c_void_p
        _host.gen_rows_host.argtypes = [ctypes.c_uint64, P, ctypes.c_int64, P, ctypes.c_int32, ctypes.c_int32, P]
        _host.gen_trace_host.argtypes = [ctypes.c_uint64, P, ctypes.c_int64, ctypes.c_int64, P, ctypes.c_uint64,
                                         ctypes.c_int32, P, ctypes.c_int32, ctypes.c_int64, P, P, P]
    return _host


def dev_lib():
    global _dev
    if _dev is None:
        path = os.path.join(HERE, "libgen_dev.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        _dev = ctypes.CDLL(path)
        P = ctypes.c_void_p
        _dev.gen_rows_dev.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, P, ctypes.c_int32,
                                      ctypes.c_int32, P, P]
        _dev.gen_trace_dev.argtypes = [ctypes.c_uint64, P, ctypes.c_int64, ctypes.c_int64, P, ctypes.c_uint64,
                                       ctypes.c_int32, P, ctypes.c_int32, ctypes.c_int64, P, P, P, P]
        _dev.gen_rows_dev.restype = ctypes.c_int
        _dev.gen_trace_dev.restype = ctypes.c_int
    return _dev


def build_host():
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", os.path.join(HERE, "libgen_host.so"),
                           os.path.join(HERE, "gen_host.c")])


def build_dev(nvcc: str = "nvcc"):
    subprocess.check_call([nvcc, "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-shared",
                           "-Xcompiler", "-fPIC", "-o", os.path.join(HERE, "libgen_dev.so"),
                           os.path.join(HERE, "gen_dev.cu")])


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def rows_host(seed: int, rho, templates: np.ndarray) -> np.ndarray:
    """Counts of expanded C3 rows ``rho`` (host build)."""
    rho = np.ascontiguousarray(rho, dtype=np.uint64)
    templates = np.ascontiguousarray(templates, dtype=np.uint32)
    T, B = templates.shape
    out = np.empty((len(rho), B), np.uint32)
    _host_lib().gen_rows_host(seed, _ptr(rho), len(rho), _ptr(templates), T, B, _ptr(out))
    return out


def trace_host(tf: TraceFamily, gids, n_arr: int):
    """(arrival int64, dist int32, true_bin int16) for scenarios ``gids``, each
    n_arr arrivals, laid out contiguously (host build)."""
    gids = np.ascontiguousarray(gids, dtype=np.uint64)
    S = len(gids)
    arr = np.empty(S * n_arr, np.int64)
    dist = np.empty(S * n_arr, np.int32)
    tb = np.empty(S * n_arr, np.int16)
    _host_lib().gen_trace_host(tf.seed, _ptr(gids), S, n_arr, _ptr(tf.exp_q16), tf.base_gap, tf.fam.D,
                               _ptr(np.ascontiguousarray(tf.cum)), tf.fam.B, T0, _ptr(arr), _ptr(dist), _ptr(tb))
    return arr, dist, tb


# ----------------------------------------------------------------------------
# feedback-loop workload: input drift + profiler sampling
# ----------------------------------------------------------------------------

def drifted_trace_family(tf: TraceFamily, slow_apps: int | None = None, num: int = 3, den: int = 2) -> TraceFamily:
    """The same arrival process and applications, but the first `slow_apps`
    applications (default: half) run num/den times slower: bin i's mass moves
    to bin min(B, ceil(i num / den)) (integer remap, totals unchanged).  Its
    traces differ from tf's only in the true bins (gen_true_bin reads only
    `cum`), so a drifted trace is the base trace with later true bins swapped
    in ("arrival pattern ... change over time")."""
    import dataclasses
    D, B = tf.fam.counts.shape
    slow = D // 2 if slow_apps is None else slow_apps
    c = tf.fam.counts.astype(np.int64).copy()
    for d in range(slow):
        row = np.zeros(B, np.int64)
        for i in range(1, B + 1):
            row[min(B, -(-i * num // den)) - 1] += c[d, i - 1]
        c[d] = row
    fam = dataclasses.replace(tf.fam, name=tf.fam.name + "-drift", counts=c.astype(np.uint32))
    return dataclasses.replace(tf, fam=fam, cum=fam.cum())


def drift_trace_host(tf: TraceFamily, gids, n_arr: int, num_epochs: int, drift_epoch: int):
    """Base trace of tf whose true bins from epoch `drift_epoch` on (epoch e of a
    scenario = arrivals [floor(e n / E), floor((e+1) n / E))) come from the
    drifted family.  Returns (arrival, dist, true_bin, drifted TraceFamily)."""
    arr, dist, tb = trace_host(tf, gids, n_arr)
    tfd = drifted_trace_family(tf)
    _, dist2, tb2 = trace_host(tfd, gids, n_arr)
    assert (dist2 == dist).all()
    j0 = (drift_epoch * n_arr) // num_epochs
    tb = tb.reshape(-1, n_arr)
    tb[:, j0:] = tb2.reshape(-1, n_arr)[:, j0:]
    return arr, dist, tb.reshape(-1), tfd


def sample_mask(seed: int, n: int, rate: float) -> np.ndarray:
    """The profiler's sample of completed requests ("finished
    requests are sampled"): uint8 [n], 1 with probability `rate` (seeded)."""
    return (np.random.default_rng(seed).random(n) < rate).astype(np.uint8)
