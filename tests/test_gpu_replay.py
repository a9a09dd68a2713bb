"""GPU parity: orloj_replay_trace vs the oracle replay.

Protocol ("follow the GPU"): the oracle replays the same trace reading the
GPU's decision log; every GPU k* must lie in the oracle's tie set T (fp64
E_k >= max - 1e-5 (k_o + k_g)), and with those decisions the integer counters
must match bit for bit.  The oracle's own free-running decisions are also
compared (documented ties only).
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle
import _parity as par

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402


def _gpu_replay(store, prof, off, arr, dist, tb, slo, bucket=None, nb=None):
    S = len(slo)
    bucket = np.arange(S) if bucket is None else bucket
    nb = S if nb is None else nb
    tr = orj.Trace(wl.t(off, np.int64), wl.t(arr, np.int64), wl.t(dist, np.int32), wl.t(tb, np.int16),
                   wl.t(slo, np.int64), wl.t(bucket, np.int32), nb)
    tr.validate(store)
    pb, log = orj.replay_trace(store, prof, tr, decision_log=True)
    torch.cuda.synchronize()
    return pb.cpu().numpy(), log.cpu().numpy()


@pytest.mark.parametrize("fam", gen.C5_FAMILIES)
def test_replay_follow_mode(fam):
    """64 scenarios (all 8 SLO buckets) x 20,000 arrivals per family."""
    tf = gen.c5_trace_family(fam)
    gids, bucket, slo = gen.c5_scenarios(tf, 8)
    n = 20000
    arr, dist, tb = gen.trace_host(tf, gids, n)
    off = np.arange(len(gids) + 1, dtype=np.int64) * n
    store = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
    prof = orj.LatencyProfile(tf.profile.a, tf.profile.w)
    pb, log = _gpu_replay(store, prof, off, arr, dist, tb, slo)
    F = oracle.cdf(tf.fam.counts)
    ref = oracle.replay(F, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo, follow_log=log)
    free = oracle.replay(F, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo, want_log=True)
    st = par.check_replay_follow(ref, pb, f"C5-20k/{fam}", free=free, log_gpu=log)
    c = pb
    assert (c[:, 1] + c[:, 2] + c[:, 3] == c[:, 0]).all()
    if fam == "static":   # integer-valued E_k: no near-ties at all
        assert st["differing_choices"] == 0
        assert (free["counters"] == pb).all() and (free["log"] == log).all()


def test_spec_cases():
    with open(os.path.join(os.path.dirname(__file__), "golden", "spec_replay.json")) as f:
        cases = json.load(f)["cases"]
    B = 100
    counts = np.zeros((3, B), np.uint32)
    counts[0, 9] = 1
    counts[1, 99] = 1
    counts[2, 9] = counts[2, 99] = 1
    store = orj.HistogramStore.from_counts(counts, 1)
    prof = orj.LatencyProfile(np.zeros(4, np.int64), np.arange(1, 5))
    for case in cases:
        dist = np.array(case.get("dist", [0 if x == 10 else 1 for x in case["true_ms"]]), np.int32)
        n = len(dist)
        pb, log = _gpu_replay(store, prof, np.array([0, n]), np.array(case["arrival"]), dist,
                              np.array(case["true_ms"]), np.array([case["slo"]]))
        assert dict(zip(orj.COUNTER_FIELDS, pb[0].tolist())) == case["expect"], case["name"]


def test_replay_edges_and_shard_invariance():
    """Empty scenarios, 1-arrival scenarios, simultaneous bursts longer than the
    window, and shard invariance: two half calls accumulate into the same
    per-bucket table as one call (integer sums, T3)."""
    tf = gen.c5_trace_family("gpt")
    gids, bucket, slo = gen.c5_scenarios(tf, 4)
    S = len(gids)
    n = 3000
    arr, dist, tb = gen.trace_host(tf, gids, n)
    arr = arr.reshape(S, n)
    arr[1, :] = arr[1, 0]                     # one huge simultaneous burst
    lens = np.full(S, n)
    lens[0], lens[2] = 0, 1
    keep = np.concatenate([np.arange(s * n, s * n + lens[s]) for s in range(S)])
    arr, dist, tb = arr.reshape(-1)[keep], dist[keep], tb[keep]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    store = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
    prof = orj.LatencyProfile(tf.profile.a, tf.profile.w)
    pb, log = _gpu_replay(store, prof, off, arr, dist, tb, slo)
    ref = oracle.replay(oracle.cdf(tf.fam.counts), tf.profile.a, tf.profile.w, off, arr, dist, tb, slo,
                        follow_log=log)
    assert (ref["ties"][:, 2] == -1).all() and (pb == ref["counters"]).all()
    assert pb[0].tolist() == [0] * 7 and pb[2, 0] == 1
    # shard invariance through the per-bucket accumulation
    nb = 8
    full, _ = _gpu_replay(store, prof, off, arr, dist, tb, slo, bucket % nb, nb)
    acc = torch.zeros((nb, 7), dtype=torch.int64, device="cuda")
    for part in (np.arange(0, S, 2), np.arange(1, S, 2)):
        sub_off = np.concatenate([[0], np.cumsum(lens[part])]).astype(np.int64)
        idx = np.concatenate([np.arange(off[s], off[s + 1]) for s in part])
        tr = orj.Trace(wl.t(sub_off, np.int64), wl.t(arr[idx], np.int64), wl.t(dist[idx], np.int32),
                       wl.t(tb[idx], np.int16), wl.t(slo[part], np.int64), wl.t(bucket[part] % nb, np.int32), nb)
        orj.replay_trace(store, prof, tr, per_bucket=acc)
    torch.cuda.synchronize()
    assert (acc.cpu().numpy() == full).all()


def test_device_generator_matches_host():
    """The device trace / row generators produce exactly the host build's values."""
    fam = wl.C5Family("rdi", local_ids=np.arange(0, 2048, 97), n_arr=4000)
    arr, dist, tb = gen.trace_host(fam.tf, fam.gids, 4000)
    assert (fam.trace.arrival.cpu().numpy() == arr).all()
    assert (fam.trace.dist.cpu().numpy() == dist).all()
    assert (fam.trace.true_bin.cpu().numpy() == tb).all()
    cfg = gen.config3(Q=64, n=256, kmax=256, T=128)
    templates = wl.t(cfg.fam.counts.view(np.int32), np.int32)
    out = torch.empty((1000, 256), dtype=torch.int32, device="cuda")
    gen.dev_lib().gen_rows_dev(cfg.row_seed, 5000, 1000, templates.data_ptr(), 128, 256, out.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    host = gen.rows_host(cfg.row_seed, np.arange(5000, 6000, dtype=np.uint64), cfg.fam.counts)
    assert (out.cpu().numpy().view(np.uint32) == host).all()


def test_replay_determinism():
    fam = wl.C5Family("skipnet", local_ids=np.arange(32), n_arr=10000)
    logs = []
    for _ in range(2):
        pb, log = orj.replay_trace(fam.store, fam.profile, fam.trace, decision_log=True)
        torch.cuda.synchronize()
        logs.append((pb.cpu().numpy(), log.cpu().numpy()))
    assert (logs[0][0] == logs[1][0]).all() and (logs[0][1] == logs[1][1]).all()


@pytest.mark.parametrize("scale", [1, 256, 2048])
def test_replay_time_scale_scan_paths(scale):
    """Every time scaled by c (arrivals, SLOs, a_k, w_k): the same decisions.
    c = 2048 puts 32 durations above 2^29, so every max-plus run scan takes the
    64-bit path; c = 256 keeps the 32-bit path except where a lookahead spans
    2^29 ticks; c = 1 is the 32-bit path throughout.  Static family: integer
    E_k, so the GPU equals the oracle's free run exactly, and the decision log
    is the unscaled one."""
    tf = gen.c5_trace_family("static")
    gids, bucket, slo = gen.c5_scenarios(tf, 2)
    n = 5000
    arr, dist, tb = gen.trace_host(tf, gids, n)
    off = np.arange(len(gids) + 1, dtype=np.int64) * n
    a = tf.profile.a.astype(np.int64) * scale
    w = tf.profile.w.astype(np.int64) * scale
    assert int(a[-1]) + int(w[-1]) * tf.fam.B < (1 << 30)            # within the validated horizon
    if scale == 2048:
        assert 32 * (int(a[0]) + int(w[0]) * tf.fam.B) >= (1 << 29)  # the kernel's 64-bit scan
    store = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks * scale)
    prof = orj.LatencyProfile(a, w)
    t0 = arr.reshape(len(gids), n)[:, :1]
    arr_s = (t0 + (arr.reshape(len(gids), n) - t0) * scale).reshape(-1)  # scaled about each scenario's start
    pb, log = _gpu_replay(store, prof, off, arr_s, dist, tb, slo * scale)  # one counter row per scenario
    F = oracle.cdf(tf.fam.counts)
    free = oracle.replay(F, a, w, off, arr_s, dist, tb, slo * scale, want_log=True)
    assert (free["counters"] == pb).all()
    assert (free["log"] == log).all()
    if scale != 1:
        store1 = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
        _, log1 = _gpu_replay(store1, orj.LatencyProfile(tf.profile.a, tf.profile.w), off, arr, dist, tb, slo)
        assert (log1 == log).all()
