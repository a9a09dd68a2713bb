"""paper_2209_00159_b200 — B200-native distribution-aware batch scoring (Orloj).

Thin Python binding over the C ABI in ``include/orloj.h`` (liborloj.so, CUDA
sm_100a).  This module only marshals arguments: every step of the hot path
(store build, candidate gather, log2-domain prefix products, bin lookup,
finish probabilities, expected finish counts, argmax, trace replay) runs in the
library's kernels.  PyTorch supplies device memory, streams and process
groups.  There is no CPU fallback: a missing library raises ``OrlojError``.

Names follow the paper (PAPER.md :241-255, Eq. 3-9 :477-543) and SURVEY.md §0.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _abi
from ._abi import OrlojError, build  # noqa: F401
from .parallel import allreduce_counters, shard_blocks, shard_round_robin  # noqa: F401

COUNTER_FIELDS = ("total", "finished", "dropped", "late", "batches", "busy_ticks", "span_ticks")


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dev(t: torch.Tensor, dtype: torch.dtype, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise OrlojError(1, f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise OrlojError(1, f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise OrlojError(1, f"{name} must be contiguous")
    return t


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


# ----------------------------------------------------------------------------
# store
# ----------------------------------------------------------------------------

class HistogramStore:
    """HBM-resident log2-CDF rows, one per distribution (application or request).

    ``log2_cdf[d, i-1] = log2 F_d(tau_i)`` in fp32; built from integer counts by
    ``orloj_store_build`` (PAPER.md:377-394 per-application histograms)."""

    def __init__(self, log2_cdf: torch.Tensor, bin_ticks: int):
        self.log2_cdf = _dev(log2_cdf, torch.float32, "log2_cdf")
        if log2_cdf.dim() != 2:
            raise OrlojError(1, "log2_cdf must be [D, B]")
        self.bin_ticks = int(bin_ticks)
        self._c = _abi.Store(log2_cdf.shape[0], log2_cdf.shape[1], self.bin_ticks, log2_cdf.data_ptr())

    @property
    def num_dists(self):
        return self.log2_cdf.shape[0]

    @property
    def num_bins(self):
        return self.log2_cdf.shape[1]

    @classmethod
    def empty(cls, num_dists: int, num_bins: int, bin_ticks: int, device="cuda") -> "HistogramStore":
        return cls(torch.empty((num_dists, num_bins), dtype=torch.float32, device=device), bin_ticks)

    def build_rows(self, counts: torch.Tensor, row0: int = 0, stream=None):
        """Fill rows [row0, row0 + len(counts)) from integer counts (device
        int32/uint32 [n, B], reinterpreted as uint32).  Synchronises the stream."""
        if counts.dtype == torch.uint32:
            counts = counts.view(torch.int32)
        counts = _dev(counts, torch.int32, "counts")
        n, B = counts.shape
        if B != self.num_bins or row0 < 0 or row0 + n > self.num_dists:
            raise OrlojError(1, "counts shape / row range does not fit the store")
        out = self.log2_cdf[row0:row0 + n]
        _abi.check(_abi.lib().orloj_store_build(counts.data_ptr(), n, B, out.data_ptr(), _stream_ptr(stream)))
        return self

    @classmethod
    def from_counts(cls, counts, bin_ticks: int, device="cuda", stream=None) -> "HistogramStore":
        if isinstance(counts, np.ndarray):
            counts = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.uint32).view(np.int32))
        counts = counts.to(device)
        st = cls.empty(counts.shape[0], counts.shape[1], bin_ticks, device)
        return st.build_rows(counts, 0, stream)

    def validate(self, stream=None):
        _abi.check(_abi.lib().orloj_validate_store(ctypes.byref(self._c), _stream_ptr(stream)))

    def c(self):
        return ctypes.byref(self._c)


class Profiler:
    """Online profiler: sampled solo execution times are
    accumulated on the GPU into integer histogram counts (orloj_histogram_
    accumulate); `refresh` rebuilds the store rows from them, `reset` starts a
    new profiling window."""

    def __init__(self, num_dists: int, num_bins: int, bin_ticks: int, device="cuda"):
        self.counts = torch.zeros((num_dists, num_bins), dtype=torch.int32, device=device)
        self.bin_ticks = int(bin_ticks)

    def add(self, dist_id: torch.Tensor, solo_ticks: torch.Tensor, stream=None):
        _dev(dist_id, torch.int32, "dist_id")
        _dev(solo_ticks, torch.int64, "solo_ticks")
        if dist_id.numel() != solo_ticks.numel():
            raise OrlojError(1, "dist_id and solo_ticks must have the same length")
        D, B = self.counts.shape
        _abi.check(_abi.lib().orloj_histogram_accumulate(dist_id.data_ptr(), solo_ticks.data_ptr(), dist_id.numel(),
                                                         self.bin_ticks, self.counts.data_ptr(), D, B,
                                                         _stream_ptr(stream)))
        return self

    def add_outcomes(self, trace: "Trace", outcome: torch.Tensor, sample_mask: Optional[torch.Tensor] = None,
                     stream=None):
        """Feedback loop: the sampled completed requests of a replay
        (outcome 1 / 2 of orloj_replay_trace_epoch) add their solo times -- the
        trace's hidden true bins -- to the window (orloj_profile_outcomes)."""
        _dev(outcome, torch.uint8, "outcome")
        if sample_mask is not None:
            _dev(sample_mask, torch.uint8, "sample_mask")
        D, B = self.counts.shape
        _abi.check(_abi.lib().orloj_profile_outcomes(trace.dist.data_ptr(), trace.true_bin.data_ptr(),
                                                     outcome.data_ptr(), _ptr(sample_mask), trace.num_arrivals,
                                                     self.counts.data_ptr(), D, B, _stream_ptr(stream)))
        return self

    def reset(self):
        self.counts.zero_()
        return self

    def refresh(self, store: "HistogramStore", stream=None, min_samples: Optional[int] = None) -> "HistogramStore":
        """Rebuild every row of `store` from the current window (orloj_store_build,
        synchronises); with min_samples, only rows whose window holds that many
        samples (orloj_store_refresh, async; the other rows are kept)."""
        if min_samples is None:
            return store.build_rows(self.counts, 0, stream)
        D, B = self.counts.shape
        _abi.check(_abi.lib().orloj_store_refresh(self.counts.data_ptr(), D, B, int(min_samples),
                                                  store.log2_cdf.data_ptr(), _stream_ptr(stream)))
        return store


# ----------------------------------------------------------------------------
# latency profile (Eq. 3 generalised, A3)
# ----------------------------------------------------------------------------

class LatencyProfile:
    """a_k (offset ticks) and w_k (ticks per bin), k = 1..kmax, non-decreasing."""

    def __init__(self, offset_ticks, ticks_per_bin):
        self.a = np.ascontiguousarray(offset_ticks, dtype=np.int64)
        self.w = np.ascontiguousarray(ticks_per_bin, dtype=np.int64)
        if self.a.shape != self.w.shape or self.a.ndim != 1:
            raise OrlojError(1, "offset_ticks / ticks_per_bin must be 1-D of equal length")
        self._c = _abi.LatencyProfile(len(self.a), self.a.ctypes.data, self.w.ctypes.data)

    @classmethod
    def eq3(cls, c0_ticks: float, c1: float, bin_ticks: int, kmax: int) -> "LatencyProfile":
        """Eq. 3 on the bin grid: a_k = round(c0), w_k = round(c1 k Delta)."""
        k = np.arange(1, kmax + 1)
        return cls(np.full(kmax, int(round(c0_ticks))), np.array([int(round(c1 * kk * bin_ticks)) for kk in k]))

    @property
    def kmax(self):
        return len(self.a)

    def c(self):
        return ctypes.byref(self._c)


# ----------------------------------------------------------------------------
# queues + score / pick
# ----------------------------------------------------------------------------

@dataclass
class Queues:
    """CSR queues on the device, members in (deadline, arrival, index) order."""
    offsets: torch.Tensor    # int64 [Q+1]
    deadline: torch.Tensor   # int64 [N]
    dist: torch.Tensor       # int32 [N]
    now: torch.Tensor        # int64 [Q]
    arrival: Optional[torch.Tensor] = None  # int64 [N], validation only
    span: Optional[int] = None  # offsets[Q] - offsets[0] (host; read from the device once when not given)

    def __post_init__(self):
        _dev(self.offsets, torch.int64, "offsets")
        _dev(self.deadline, torch.int64, "deadline")
        _dev(self.dist, torch.int32, "dist")
        _dev(self.now, torch.int64, "now")
        if self.arrival is not None:
            _dev(self.arrival, torch.int64, "arrival")
        self._c = _abi.QueuesC(self.now.numel(), self.offsets.data_ptr(), _ptr(self.arrival),
                               self.deadline.data_ptr(), self.dist.data_ptr(), self.now.data_ptr())

    @property
    def num_queues(self):
        return self.now.numel()

    @property
    def members(self) -> int:
        """Members covered by the offsets, offsets[Q] - offsets[0]: the row length
        of the [S][N] priority outputs (the offsets may start at any base)."""
        if self.span is None:
            self.span = int(self.offsets[-1].item() - self.offsets[0].item())
        return self.span

    @classmethod
    def from_numpy(cls, offsets, deadline, dist, now, arrival=None, device="cuda") -> "Queues":
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device)  # noqa: E731
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        return cls(t(off, np.int64), t(deadline, np.int64), t(dist, np.int32), t(now, np.int64),
                   None if arrival is None else t(arrival, np.int64), int(off[-1] - off[0]))

    def validate(self, store: HistogramStore, stream=None):
        _abi.check(_abi.lib().orloj_validate_queues(store.c(), ctypes.byref(self._c), _stream_ptr(stream)))

    def c(self):
        return ctypes.byref(self._c)


def score_batches(store: HistogramStore, profile: LatencyProfile, queues: Queues, want_P: bool = False,
                  want_EL: bool = False, stream=None, out: Optional[dict] = None) -> dict:
    """E_k for every candidate prefix (+ optional P_r(k), E[L_{B_k}]).  Async on `stream`."""
    Q, kmax = queues.num_queues, profile.kmax
    dev = queues.now.device
    out = out or {}
    E = out.get("E")
    if E is None:
        E = torch.empty((Q, kmax), dtype=torch.float32, device=dev)
    P = out.get("P") if want_P else None
    if want_P and P is None:
        P = torch.zeros((Q, kmax * (kmax + 1) // 2), dtype=torch.float32, device=dev)
    EL = out.get("EL") if want_EL else None
    if want_EL and EL is None:
        EL = torch.empty((Q, kmax), dtype=torch.float32, device=dev)
    _abi.check(_abi.lib().orloj_score_batches(store.c(), profile.c(), queues.c(), E.data_ptr(), _ptr(P),
                                              _ptr(EL), _stream_ptr(stream)))
    return {"E": E, "P": P, "EL": EL}


def pick_batch(store: HistogramStore, profile: LatencyProfile, queues: Queues, best_k=None, best_E=None,
               stream=None):
    """k* = smallest argmax_k E_k per queue (0 for empty queues) and E_{k*}.  Async."""
    Q = queues.num_queues
    dev = queues.now.device
    if best_k is None:
        best_k = torch.empty(Q, dtype=torch.int32, device=dev)
    if best_E is None:
        best_E = torch.empty(Q, dtype=torch.float32, device=dev)
    _abi.check(_abi.lib().orloj_pick_batch(store.c(), profile.c(), queues.c(), best_k.data_ptr(),
                                           best_E.data_ptr(), _stream_ptr(stream)))
    return best_k, best_E


class PriorityTable:
    """Eq. 1-2 priorities for batch sizes 1..num_sizes, with
    the batch-latency distribution of each size from the mixture of all
    applications, precomputed off the critical path
    (orloj_priority_table); `scores` evaluates log p for every queue member and
    size, `pop` selects the top members of a size per queue (PopBatch)."""

    def __init__(self, store: HistogramStore, profile: LatencyProfile, num_sizes: int, b_per_tick: float,
                 weights: Optional[torch.Tensor] = None, stream=None):
        dev = store.log2_cdf.device
        self.store, self.profile = store, profile
        self.S, self.b = int(num_sizes), float(b_per_tick)
        self.log_table = torch.empty((self.S, 2, store.num_bins + 1), dtype=torch.float64, device=dev)
        self.log_expected = torch.empty(self.S, dtype=torch.float64, device=dev)
        if weights is not None:
            _dev(weights, torch.float32, "weights")
        _abi.check(_abi.lib().orloj_priority_table(store.c(), profile.c(), self.S, _ptr(weights), self.b,
                                                   self.log_table.data_ptr(), self.log_expected.data_ptr(),
                                                   _stream_ptr(stream)))

    def scores(self, queues: Queues, out: Optional[torch.Tensor] = None, stream=None, steps=None) -> torch.Tensor:
        """log p [S][N].  steps = (offset_ticks, cumulative_costs): piecewise-step
        cost, deadlines D_r + offset with cost c_s after each."""
        N = queues.members  # row length: offsets[Q] - offsets[0] (the kernel's [S][N] layout)
        if out is None:
            out = torch.empty((self.S, N), dtype=torch.float32, device=queues.now.device)
        elif out.numel() < self.S * N:
            raise OrlojError(1, f"out must hold num_sizes x {N} floats")
        if steps is None:
            _abi.check(_abi.lib().orloj_priority_scores(self.store.c(), self.profile.c(), self.S, self.b,
                                                        self.log_table.data_ptr(), self.log_expected.data_ptr(),
                                                        queues.c(), _ptr(out), _stream_ptr(stream)))
        else:
            off = np.ascontiguousarray(steps[0], dtype=np.int64)
            cost = np.ascontiguousarray(steps[1], dtype=np.float64)
            if off.shape != cost.shape or off.ndim != 1:
                raise OrlojError(1, "steps: offsets and costs must be 1-D of equal length")
            cs = _abi.CostSteps(len(off), off.ctypes.data, cost.ctypes.data)
            _abi.check(_abi.lib().orloj_priority_scores_steps(self.store.c(), self.profile.c(), self.S, self.b,
                                                              self.log_table.data_ptr(), self.log_expected.data_ptr(),
                                                              queues.c(), ctypes.byref(cs), _ptr(out),
                                                              _stream_ptr(stream)))
        return out

    def pop(self, queues: Queues, log_priority: torch.Tensor, batch_size: torch.Tensor, stream=None,
            out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Selected member indices [Q][32] (-1 padded) for the [S][N] scores."""
        _dev(log_priority, torch.float32, "log_priority")
        _dev(batch_size, torch.int32, "batch_size")
        if log_priority.dim() != 2 or log_priority.shape[0] != self.S:
            raise OrlojError(1, "log_priority must be [num_sizes, N]")
        sel = out if out is not None else torch.empty((queues.num_queues, 32), dtype=torch.int32,
                                                      device=queues.now.device)
        _abi.check(_abi.lib().orloj_pop_batch(queues.c(), log_priority.data_ptr(), self.S, batch_size.data_ptr(),
                                              _ptr(sel), _stream_ptr(stream)))
        return sel


class ScoreModel:
    """Scoring-model variant (orloj_score_model_batches):
    a duration table dur[k-1][m] (m = 0..B) instead of the Eq. 3 profile,
    upper-edge or within-bin-uniform bins, and a piecewise-step cost (weighted
    finish count).  kmax <= 32, B <= 128."""

    def __init__(self, duration_ticks, interpolate: bool = False, steps=None, device="cuda"):
        dur = np.ascontiguousarray(duration_ticks, dtype=np.int64)
        if dur.ndim != 2 or not 1 <= dur.shape[0] <= 32:
            raise OrlojError(1, "duration table must be [kmax <= 32, B+1]")
        if (np.diff(dur, axis=1) < 0).any():
            raise OrlojError(1, "duration table must be non-decreasing in the bin position")
        self.kmax, self.num_bins = dur.shape[0], dur.shape[1] - 1
        self.dur_host = dur
        self.dur = torch.from_numpy(dur).to(device)
        self.interpolate = bool(interpolate)
        if steps is None:
            self.off = np.zeros(0, np.int64)
            self.cost = np.zeros(0, np.float64)
        else:
            self.off = np.ascontiguousarray(steps[0], dtype=np.int64)
            self.cost = np.ascontiguousarray(steps[1], dtype=np.float64)
            if self.off.shape != self.cost.shape or self.off.ndim != 1:
                raise OrlojError(1, "steps: offsets and costs must be 1-D of equal length")
        # the table's row analysis, once (orloj_score_model_prepare), reused by every score call
        self.plan = torch.empty(_abi.SCORE_MODEL_PLAN_BYTES, dtype=torch.uint8, device=self.dur.device)
        self._c = _abi.ScoreModelC(self.kmax, self.dur.data_ptr(), int(self.interpolate), 0, None, None, None)
        _abi.check(_abi.lib().orloj_score_model_prepare(ctypes.byref(self._c), self.num_bins, self.plan.data_ptr(),
                                                        _stream_ptr(None)))
        torch.cuda.current_stream(self.dur.device).synchronize()  # the plan is read on any stream later

    @classmethod
    def eq3(cls, profile: "LatencyProfile", num_bins: int, **kw) -> "ScoreModel":
        """The main scorer's model: dur[k-1][m] = a_k + w_k m."""
        m = np.arange(num_bins + 1, dtype=np.int64)
        return cls(profile.a[:, None] + profile.w[:, None] * m[None, :], **kw)

    def c(self):
        self._c = _abi.ScoreModelC(self.kmax, self.dur.data_ptr(), int(self.interpolate), len(self.off),
                                   self.off.ctypes.data if len(self.off) else None,
                                   self.cost.ctypes.data if len(self.cost) else None, self.plan.data_ptr())
        return ctypes.byref(self._c)

    def score(self, store: HistogramStore, queues: Queues, stream=None, out: Optional[dict] = None) -> dict:
        """E [Q][kmax], best_k [Q], best_E [Q].  Async on `stream`."""
        if store.num_bins != self.num_bins:
            raise OrlojError(1, "duration table and store disagree on B")
        Q, dev = queues.num_queues, queues.now.device
        out = out or {}
        E = out.get("E") if out.get("E") is not None else torch.empty((Q, self.kmax), dtype=torch.float32, device=dev)
        bk = out.get("best_k") if out.get("best_k") is not None else torch.empty(Q, dtype=torch.int32, device=dev)
        bE = out.get("best_E") if out.get("best_E") is not None else torch.empty(Q, dtype=torch.float32, device=dev)
        _abi.check(_abi.lib().orloj_score_model_batches(store.c(), queues.c(), self.c(), E.data_ptr(), bk.data_ptr(),
                                                        bE.data_ptr(), _stream_ptr(stream)))
        return {"E": E, "best_k": bk, "best_E": bE}


class HostPicker:
    """End-to-end pick for queues in pinned host memory (orloj_pick_batch_host).

    The queue set is cut into `chunks` contiguous chunks issued round-robin on
    `streams` CUDA streams, each with its own device workspace: every call
    enqueues its chunk's H2D copies, the pick kernel and the D2H copies of the
    results, so the copy of chunk c+1 overlaps the kernel of chunk c (the copy
    engine and the SMs run concurrently).  `pick` returns after enqueueing and
    making the caller's stream wait for every chunk."""

    def __init__(self, store: HistogramStore, profile: LatencyProfile, offsets, chunks: int = 1,
                 streams: int = 1, device="cuda"):
        self.store, self.profile = store, profile
        off = np.asarray(offsets, dtype=np.int64)
        self.Q, self.N = len(off) - 1, int(off[-1] - off[0])
        chunks = max(1, min(int(chunks), max(self.Q, 1)))
        qb = np.linspace(0, self.Q, chunks + 1).astype(np.int64)
        self.bounds = [(int(a), int(b), int(off[a] - off[0]), int(off[b] - off[0])) for a, b in zip(qb[:-1], qb[1:])]
        self.streams = [torch.cuda.Stream(device) for _ in range(max(1, int(streams)))]
        self.ws = []
        for i in range(len(self.streams)):
            need = max(_abi.lib().orloj_pick_batch_host_workspace(b - a, m1 - m0)
                       for j, (a, b, m0, m1) in enumerate(self.bounds) if j % len(self.streams) == i) \
                if len(self.bounds) > i else 256
            buf = torch.empty(need + 256, dtype=torch.uint8, device=device)
            self.ws.append((buf, (buf.data_ptr() + 255) & ~255, need))
        self.best_k = torch.empty(self.Q, dtype=torch.int32).pin_memory()
        self.best_E = torch.empty(self.Q, dtype=torch.float32).pin_memory()

    def h2d_bytes(self):
        return sum((b - a + 1) * 8 + (m1 - m0) * 12 + (b - a) * 8 for a, b, m0, m1 in self.bounds)

    def d2h_bytes(self):
        return self.Q * 8

    def pick(self, offsets: torch.Tensor, deadline: torch.Tensor, dist: torch.Tensor, now: torch.Tensor,
             stream=None):
        for t, dt, n in ((offsets, torch.int64, "offsets"), (deadline, torch.int64, "deadline"),
                         (dist, torch.int32, "dist"), (now, torch.int64, "now")):
            if t.is_cuda or t.dtype != dt or not t.is_contiguous():
                raise OrlojError(1, f"{n} must be a contiguous host {dt} tensor (pinned for async copies)")
        main = stream or torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(main)
        for s in self.streams:
            s.wait_event(start)
        L = _abi.lib()
        for j, (a, b, m0, m1) in enumerate(self.bounds):
            s = self.streams[j % len(self.streams)]
            _, ws, wsb = self.ws[j % len(self.streams)]
            _abi.check(L.orloj_pick_batch_host(
                self.store.c(), self.profile.c(), b - a, offsets.data_ptr() + 8 * a, deadline.data_ptr() + 8 * m0,
                dist.data_ptr() + 4 * m0, now.data_ptr() + 8 * a, self.best_k.data_ptr() + 4 * a,
                self.best_E.data_ptr() + 4 * a, ws, wsb, s.cuda_stream))
        for s in self.streams:
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
        return self.best_k, self.best_E


# ----------------------------------------------------------------------------
# trace replay
# ----------------------------------------------------------------------------

@dataclass
class Trace:
    """Arrival trace of many independent scenarios (CSR), constant SLO each."""
    offsets: torch.Tensor    # int64 [S+1]
    arrival: torch.Tensor    # int64 [N]
    dist: torch.Tensor       # int32 [N]
    true_bin: torch.Tensor   # int16 [N]
    slo: torch.Tensor        # int64 [S]
    bucket: torch.Tensor     # int32 [S]
    num_buckets: int

    def __post_init__(self):
        _dev(self.offsets, torch.int64, "offsets")
        _dev(self.arrival, torch.int64, "arrival")
        _dev(self.dist, torch.int32, "dist")
        _dev(self.true_bin, torch.int16, "true_bin")
        _dev(self.slo, torch.int64, "slo")
        _dev(self.bucket, torch.int32, "bucket")
        if self.offsets.numel() != self.slo.numel() + 1:
            raise OrlojError(1, "offsets must have num_scenarios + 1 entries")
        # the segmented replay sizes its scratch from num_arrivals = arrival.numel()
        if self.slo.numel() > 0 and int(self.offsets[-1]) != self.arrival.numel():
            raise OrlojError(1, "offsets[-1] must equal the number of arrivals")
        self._c = _abi.TraceC(self.slo.numel(), self.offsets.data_ptr(), self.arrival.data_ptr(),
                              self.dist.data_ptr(), self.true_bin.data_ptr(), self.slo.data_ptr(),
                              self.bucket.data_ptr(), int(self.num_buckets))

    @property
    def num_scenarios(self):
        return self.slo.numel()

    @property
    def num_arrivals(self):
        return self.arrival.numel()

    def validate(self, store: HistogramStore, stream=None):
        _abi.check(_abi.lib().orloj_validate_trace(store.c(), ctypes.byref(self._c), _stream_ptr(stream)))

    def c(self):
        return ctypes.byref(self._c)


OBJECTIVES = {"expected_finish": 0, "finish_rate": 1, "alg1": 2}


def replay_trace(store: HistogramStore, profile: LatencyProfile, trace: Trace, per_bucket=None,
                 decision_log: bool | torch.Tensor = False, stream=None, objective: str = "expected_finish",
                 drop_threshold: Optional[torch.Tensor] = None, priority: Optional["PriorityTable"] = None,
                 size_thresholds: Optional[torch.Tensor] = None, segments: int = 1,
                 workspace: Optional[torch.Tensor] = None):
    """Replay every scenario; returns (per_bucket int64 [num_buckets, 7], log or None).
    per_bucket is ADDED to (pass a zeroed tensor to accumulate across calls).
    objective: "expected_finish" (argmax E_k) or "finish_rate" (argmax
    E_k / E[L_{B_k}]); drop_threshold: device int64 [num_dists] (see
    policy.expected_latency_thresholds) or None for the hopeless rule.
    objective "alg1" (the paper's Alg. 1 iteration, include/orloj.h) needs
    `priority` (a PriorityTable with num_sizes = kmax) and `size_thresholds`
    (device int64 [kmax], policy.alg1_size_thresholds); the decision log then
    holds popped-member bit masks.
    segments > 1: the exact segmented replay (orloj_replay_trace_seg; same
    counters and log, shorter critical path); `workspace` (uint8 device tensor
    of replay_seg_workspace_bytes(...) bytes) is allocated when not given."""
    dev = trace.arrival.device
    if per_bucket is None:
        per_bucket = torch.zeros((trace.num_buckets, 7), dtype=torch.int64, device=dev)
    _dev(per_bucket, torch.int64, "per_bucket")
    log = None
    if isinstance(decision_log, torch.Tensor):
        log = _dev(decision_log, torch.int32, "decision_log")
    elif decision_log:
        log = torch.zeros(trace.num_arrivals + trace.num_scenarios, dtype=torch.int32, device=dev)
    if objective not in OBJECTIVES:
        raise OrlojError(1, f"objective must be one of {sorted(OBJECTIVES)}")
    if drop_threshold is not None:
        _dev(drop_threshold, torch.int64, "drop_threshold")
        if drop_threshold.numel() != store.num_dists:
            raise OrlojError(1, "drop_threshold must have one entry per distribution")
    pol = _abi.ReplayPolicyC(OBJECTIVES[objective], _ptr(drop_threshold), None, None, None, 0.0)
    if objective == "alg1":
        if priority is None or size_thresholds is None:
            raise OrlojError(1, "objective alg1 needs priority tables and size thresholds")
        if priority.S != profile.kmax:
            raise OrlojError(1, "alg1: the priority tables must cover batch sizes 1..kmax")
        _dev(size_thresholds, torch.int64, "size_thresholds")
        if size_thresholds.numel() != profile.kmax:
            raise OrlojError(1, "size_thresholds must have kmax entries")
        pol.size_threshold_ticks = size_thresholds.data_ptr()
        pol.priority_table = priority.log_table.data_ptr()
        pol.priority_log_expected = priority.log_expected.data_ptr()
        pol.priority_b_per_tick = priority.b
    if segments == 1:
        _abi.check(_abi.lib().orloj_replay_trace_ex(store.c(), profile.c(), trace.c(), ctypes.byref(pol),
                                                    per_bucket.data_ptr(), _ptr(log), _stream_ptr(stream)))
        return per_bucket, log
    need = replay_seg_workspace_bytes(trace, segments, log is not None)
    if workspace is None:
        workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
    _dev(workspace, torch.uint8, "workspace")
    _abi.check(_abi.lib().orloj_replay_trace_seg(store.c(), profile.c(), trace.c(), ctypes.byref(pol), int(segments),
                                                 trace.num_arrivals, _ptr(workspace), workspace.numel(),
                                                 per_bucket.data_ptr(), _ptr(log), _stream_ptr(stream)))
    return per_bucket, log


OUTCOME = {1: "finished", 2: "late", 3: "dropped"}


def replay_epoch(store: HistogramStore, profile: LatencyProfile, trace: Trace, epoch: int, num_epochs: int,
                 worker_free: Optional[torch.Tensor] = None, outcome: Optional[torch.Tensor] = None,
                 per_bucket=None, decision_log: bool | torch.Tensor = False, stream=None):
    """One epoch of a replay cut into num_epochs (orloj_replay_trace_epoch):
    arrivals [floor(e n / E), floor((e+1) n / E)) of each scenario, the worker
    busy until worker_free[s] (int64 [S], updated in place; fill with
    INT64_MIN for a free worker), per-arrival outcomes into `outcome` (uint8
    [N]: 1 finished, 2 late, 3 dropped).  Returns (per_bucket, log or None)."""
    dev = trace.arrival.device
    if per_bucket is None:
        per_bucket = torch.zeros((trace.num_buckets, 7), dtype=torch.int64, device=dev)
    _dev(per_bucket, torch.int64, "per_bucket")
    if worker_free is not None:
        _dev(worker_free, torch.int64, "worker_free")
        if worker_free.numel() != trace.num_scenarios:
            raise OrlojError(1, "worker_free must have one entry per scenario")
    if outcome is not None:
        _dev(outcome, torch.uint8, "outcome")
        if outcome.numel() != trace.num_arrivals:
            raise OrlojError(1, "outcome must have one entry per arrival")
    log = None
    if isinstance(decision_log, torch.Tensor):
        log = _dev(decision_log, torch.int32, "decision_log")
    elif decision_log:
        log = torch.zeros(trace.num_arrivals + trace.num_scenarios, dtype=torch.int32, device=dev)
    ep = _abi.ReplayEpochC(int(epoch), int(num_epochs), _ptr(worker_free), _ptr(outcome))
    _abi.check(_abi.lib().orloj_replay_trace_epoch(store.c(), profile.c(), trace.c(), None, ctypes.byref(ep),
                                                   per_bucket.data_ptr(), _ptr(log), _stream_ptr(stream)))
    return per_bucket, log


def replay_feedback(store: HistogramStore, profile: LatencyProfile, trace: Trace, num_epochs: int,
                    window_epochs: int, min_samples: int = 1, sample_mask: Optional[torch.Tensor] = None,
                    decision_logs: bool = False, stream=None) -> dict:
    """The long-term feedback loop (orloj_replay_feedback):
    epochs replayed with the current store, sampled completed requests
    profiled, rows with >= min_samples window samples rebuilt in place in
    `store`, the window reset every window_epochs epochs.  Returns dict(
    per_epoch int64 [E, num_buckets, 7], window uint32-as-int32 [D, B] (the
    window of the last refresh), logs int32 [E, N + S] or None)."""
    dev = trace.arrival.device
    E = int(num_epochs)
    if sample_mask is not None:
        _dev(sample_mask, torch.uint8, "sample_mask")
        if sample_mask.numel() != trace.num_arrivals:
            raise OrlojError(1, "sample_mask must have one entry per arrival")
    per_epoch = torch.zeros((E, trace.num_buckets, 7), dtype=torch.int64, device=dev)
    window = torch.zeros((store.num_dists, store.num_bins), dtype=torch.int32, device=dev)
    logs = (torch.zeros((E, trace.num_arrivals + trace.num_scenarios), dtype=torch.int32, device=dev)
            if decision_logs else None)
    L = _abi.lib()
    need = int(L.orloj_replay_feedback_workspace(trace.num_scenarios, trace.num_arrivals, store.num_dists,
                                                 store.num_bins))
    buf = torch.empty(need + 256, dtype=torch.uint8, device=dev)
    ws = (buf.data_ptr() + 255) & ~255
    fb = _abi.FeedbackC(E, int(window_epochs), int(min_samples), _ptr(sample_mask))
    _abi.check(L.orloj_replay_feedback(store.c(), profile.c(), trace.c(), None, ctypes.byref(fb), ws, need,
                                       per_epoch.data_ptr(), window.data_ptr(), _ptr(logs), _stream_ptr(stream)))
    # the workspace is returned so it outlives the asynchronous work on `stream`
    return {"per_epoch": per_epoch, "window": window, "logs": logs, "_workspace": buf}


def replay_seg_stats(workspace: torch.Tensor) -> dict:
    """Diagnostics a completed segmented replay left in its workspace head."""
    v = workspace[:40].view(torch.int64).cpu().tolist()
    return {"stitch_decisions": v[0], "joined": v[1], "crossed": v[2], "extension_decisions": v[3],
            "size_error": v[4]}


def replay_seg_workspace_bytes(trace: Trace, segments: int, with_log: bool = False) -> int:
    """Device workspace of the segmented replay (orloj_replay_seg_workspace)."""
    return int(_abi.lib().orloj_replay_seg_workspace(trace.num_scenarios, trace.num_arrivals, int(segments),
                                                     int(bool(with_log))))
