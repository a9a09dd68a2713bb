"""Device-side workload setup shared by bench.py and the GPU tests.

Plumbing only: seeded inputs come from ``gen`` (data, no method arithmetic);
every step of the hot path runs through the public API of
``paper_2209_00159_b200`` (C ABI -> CUDA).  Nothing here touches ``oracle``.
"""
from __future__ import annotations

import numpy as np
import torch

import gen
import paper_2209_00159_b200 as orj


def t(a, dtype, device="cuda"):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(device)


def c3_store(cfg: gen.ScoreConfig, device="cuda", chunk_rows: int = 1 << 20, stream=None) -> orj.HistogramStore:
    """Per-request rows of C3: expanded from integer templates on the device
    (gen_dev.cu) chunk by chunk, then turned into log2-CDF rows by
    orloj_store_build."""
    B = cfg.fam.B
    templates = t(cfg.fam.counts.view(np.int32), np.int32, device)
    store = orj.HistogramStore.empty(cfg.n_rows, B, cfg.fam.bin_ticks, device)
    counts = torch.empty((min(chunk_rows, cfg.n_rows), B), dtype=torch.int32, device=device)
    lib = gen.dev_lib()
    sp = torch.cuda.current_stream().cuda_stream if stream is None else stream.cuda_stream
    for r0 in range(0, cfg.n_rows, chunk_rows):
        n = min(chunk_rows, cfg.n_rows - r0)
        st = lib.gen_rows_dev(cfg.row_seed, r0, n, templates.data_ptr(), templates.shape[0], B,
                              counts.data_ptr(), sp)
        assert st == 0, f"gen_rows_dev failed ({st})"
        store.build_rows(counts[:n], r0, stream)
    del counts
    return store


def score_store(cfg: gen.ScoreConfig, device="cuda") -> orj.HistogramStore:
    if cfg.rows == "c3":
        return c3_store(cfg, device)
    return orj.HistogramStore.from_counts(cfg.fam.counts, cfg.fam.bin_ticks, device)


def device_queues(q: gen.Queues, device="cuda", with_arrival=True) -> orj.Queues:
    return orj.Queues.from_numpy(q.offsets, q.deadline, q.dist, q.now, q.arrival if with_arrival else None, device)


def profile(p: gen.Profile) -> orj.LatencyProfile:
    return orj.LatencyProfile(p.a, p.w)


class C5Family:
    """One family of the C5 sweep on the device: store, profile, trace."""

    def __init__(self, name: str, local_ids=None, n_arr: int = gen.C5_ARRIVALS,
                 seeds_per_bucket: int = gen.C5_SEEDS_PER_BUCKET, device="cuda", on_host=False, drift=None):
        """drift = (num_epochs, drift_epoch): true bins from epoch drift_epoch on
        come from gen.drifted_trace_family (feedback-loop workload)."""
        self.tf = gen.c5_trace_family(name)
        gids, bucket, slo = gen.c5_scenarios(self.tf, seeds_per_bucket)
        if local_ids is not None:
            gids, bucket, slo = gids[local_ids], bucket[local_ids], slo[local_ids]
        self.gids, self.bucket_np, self.slo_np = gids, bucket, slo
        S = len(gids)
        self.n_arr = n_arr
        self.offsets_np = np.arange(S + 1, dtype=np.int64) * n_arr
        self.store = orj.HistogramStore.from_counts(self.tf.fam.counts, self.tf.fam.bin_ticks, device)
        self.profile = orj.LatencyProfile(self.tf.profile.a, self.tf.profile.w)
        if on_host:
            arr, dist, tb = gen.trace_host(self.tf, gids, n_arr)
            arrival, dist_t, tb_t = t(arr, np.int64, device), t(dist, np.int32, device), t(tb, np.int16, device)
        else:
            N = S * n_arr
            arrival = torch.empty(N, dtype=torch.int64, device=device)
            dist_t = torch.empty(N, dtype=torch.int32, device=device)
            tb_t = torch.empty(N, dtype=torch.int16, device=device)
            g = t(gids.view(np.int64), np.int64, device)
            e = t(self.tf.exp_q16.view(np.int32), np.int32, device)
            cum = t(self.tf.cum.view(np.int32), np.int32, device)
            st = gen.dev_lib().gen_trace_dev(self.tf.seed, g.data_ptr(), S, n_arr, e.data_ptr(), self.tf.base_gap,
                                             self.tf.fam.D, cum.data_ptr(), self.tf.fam.B, gen.T0,
                                             arrival.data_ptr(), dist_t.data_ptr(), tb_t.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream)
            assert st == 0, f"gen_trace_dev failed ({st})"
            if drift is not None:
                E, e0 = drift
                self.tfd = gen.drifted_trace_family(self.tf)
                cum2 = t(self.tfd.cum.view(np.int32), np.int32, device)
                a2 = torch.empty_like(arrival)
                d2 = torch.empty_like(dist_t)
                tb2 = torch.empty_like(tb_t)
                st = gen.dev_lib().gen_trace_dev(self.tf.seed, g.data_ptr(), S, n_arr, e.data_ptr(),
                                                 self.tf.base_gap, self.tf.fam.D, cum2.data_ptr(), self.tf.fam.B,
                                                 gen.T0, a2.data_ptr(), d2.data_ptr(), tb2.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream)
                assert st == 0, f"gen_trace_dev failed ({st})"
                j0 = (e0 * n_arr) // E
                tb_t.view(S, n_arr)[:, j0:] = tb2.view(S, n_arr)[:, j0:]
                del a2, d2, tb2
        self.trace = orj.Trace(t(self.offsets_np, np.int64, device), arrival, dist_t, tb_t,
                               t(slo, np.int64, device), t(bucket, np.int32, device), len(gen.BUCKET_SLO_MULTS))

    @property
    def num_scenarios(self):
        return len(self.gids)
