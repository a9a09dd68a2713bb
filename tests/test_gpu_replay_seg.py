"""GPU parity of the segmented replay (orloj_replay_trace_seg, include/orloj.h):
speculative segments stitched at regeneration points must give the plain
replay's counters and decision log bit for bit, for every policy, segment
count and the degenerate traces (empty / one-arrival scenarios, bursts with no
regeneration point, more segments than arrivals); and the oracle, following
the segmented log, reproduces the counters."""
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
from paper_2209_00159_b200 import policy  # noqa: E402


def _family(fam, seeds, n):
    tf = gen.c5_trace_family(fam)
    gids, bucket, slo = gen.c5_scenarios(tf, seeds)
    arr, dist, tb = gen.trace_host(tf, gids, n)
    off = np.arange(len(gids) + 1, dtype=np.int64) * n
    return tf, off, arr, dist, tb, slo


def _trace(off, arr, dist, tb, slo):
    S = len(slo)
    return orj.Trace(wl.t(off, np.int64), wl.t(arr, np.int64), wl.t(dist, np.int32), wl.t(tb, np.int16),
                     wl.t(slo, np.int64), wl.t(np.arange(S), np.int32), S)


def _kw(tf, store, prof, objective, drop):
    kw = dict(objective=objective)
    if drop == "expected_latency":
        kw["drop_threshold"] = wl.t(policy.expected_latency_thresholds(tf.fam.counts, tf.profile.a, tf.profile.w),
                                    np.int64)
    if objective == "alg1":
        a, w = tf.profile.a, tf.profile.w
        kw["priority"] = orj.PriorityTable(store, prof, len(a), 1.0 / float(np.mean(a + w * 8)))
        kw["size_thresholds"] = wl.t(policy.alg1_size_thresholds(tf.fam.counts, a, w), np.int64)
    return kw


def _both(store, prof, tr, segments, **kw):
    pb0, log0 = orj.replay_trace(store, prof, tr, decision_log=True, **kw)
    pb1, log1 = orj.replay_trace(store, prof, tr, decision_log=True, segments=segments, **kw)
    pb2, _ = orj.replay_trace(store, prof, tr, segments=segments, **kw)  # without a log
    torch.cuda.synchronize()
    return pb0.cpu().numpy(), log0.cpu().numpy(), pb1.cpu().numpy(), log1.cpu().numpy(), pb2.cpu().numpy()


@pytest.mark.parametrize("fam", gen.C5_FAMILIES)
@pytest.mark.parametrize("objective,drop", [("expected_finish", "hopeless"), ("finish_rate", "expected_latency"),
                                            ("alg1", "hopeless")])
def test_segmented_equals_plain(fam, objective, drop):
    """32 scenarios (all 8 SLO buckets) x 20,000 arrivals; 2, 7 and 64 segments."""
    tf, off, arr, dist, tb, slo = _family(fam, 4, 20000)
    store = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
    prof = orj.LatencyProfile(tf.profile.a, tf.profile.w)
    tr = _trace(off, arr, dist, tb, slo)
    kw = _kw(tf, store, prof, objective, drop)
    for G in (2, 7, 64):
        pb0, log0, pb1, log1, pb2 = _both(store, prof, tr, G, **kw)
        assert (pb1 == pb0).all(), (G, np.argwhere(pb1 != pb0)[:5])
        assert (pb2 == pb0).all(), G
        assert (log1 == log0).all(), (G, np.flatnonzero(log1 != log0)[:5])


def test_segmented_follow_oracle():
    """The oracle follows the segmented replay's log: decisions in its tie sets,
    counters bit-exact."""
    tf, off, arr, dist, tb, slo = _family("skipnet", 8, 20000)
    store = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
    prof = orj.LatencyProfile(tf.profile.a, tf.profile.w)
    pb, log = orj.replay_trace(store, prof, _trace(off, arr, dist, tb, slo), decision_log=True, segments=16)
    torch.cuda.synchronize()
    pb, log = pb.cpu().numpy(), log.cpu().numpy()
    ref = oracle.replay(oracle.cdf(tf.fam.counts), tf.profile.a, tf.profile.w, off, arr, dist, tb, slo,
                        follow_log=log)
    par.check_replay_follow(ref, pb, "segmented-16/skipnet")
    assert (pb[:, 1] + pb[:, 2] + pb[:, 3] == pb[:, 0]).all()


def test_segmented_edges():
    """Empty and one-arrival scenarios, a simultaneous burst (no regeneration
    point until it drains: the stitch runs through every segment), a trace of
    back-to-back overload, and more segments than arrivals."""
    tf = gen.c5_trace_family("gpt")
    gids, bucket, slo = gen.c5_scenarios(tf, 2)
    S = len(gids)
    n = 3000
    arr, dist, tb = gen.trace_host(tf, gids, n)
    arr = arr.reshape(S, n)
    arr[1, :] = arr[1, 0]                                     # one huge simultaneous burst
    arr[3, :] = arr[3, 0] + np.arange(n) * 10                 # arrivals far faster than service
    lens = np.full(S, n)
    lens[0], lens[2], lens[5] = 0, 1, 33
    keep = np.concatenate([np.arange(s * n, s * n + lens[s]) for s in range(S)])
    arr, dist, tb = arr.reshape(-1)[keep], dist[keep], tb[keep]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    store = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
    prof = orj.LatencyProfile(tf.profile.a, tf.profile.w)
    tr = _trace(off, arr, dist, tb, slo)
    for G in (2, 3, 31, 4096):
        pb0, log0, pb1, log1, pb2 = _both(store, prof, tr, G)
        assert (pb1 == pb0).all() and (pb2 == pb0).all() and (log1 == log0).all(), G
    assert pb0[0].tolist() == [0] * 7 and pb0[2, 0] == 1


def test_segmented_arguments():
    tf, off, arr, dist, tb, slo = _family("static", 1, 100)
    store = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
    prof = orj.LatencyProfile(tf.profile.a, tf.profile.w)
    tr = _trace(off, arr, dist, tb, slo)
    need = orj.replay_seg_workspace_bytes(tr, 4)
    assert need > 0 and orj.replay_seg_workspace_bytes(tr, 1) == 0
    assert orj.replay_seg_workspace_bytes(tr, 4, True) > need
    small = torch.empty(need - 256, dtype=torch.uint8, device="cuda")
    with pytest.raises(orj.OrlojError, match="workspace"):
        orj.replay_trace(store, prof, tr, segments=4, workspace=small)
    with pytest.raises(orj.OrlojError, match="segments"):
        orj.replay_trace(store, prof, tr, segments=0)
    with pytest.raises(orj.OrlojError, match="segments"):
        orj.replay_trace(store, prof, tr, segments=5000)


@pytest.mark.parametrize("B", [16, 100])
def test_segmented_other_bin_widths(B):
    """Bins-per-lane variants 1 and 4 (the C5 families use 64 bins): random
    histograms and a random bursty trace, segmented == plain."""
    rng = np.random.default_rng(B)
    D, S, n = 5, 12, 4000
    counts = rng.integers(0, 50, size=(D, B)).astype(np.uint32)
    counts[:, -1] += 1
    store = orj.HistogramStore.from_counts(counts, 10)
    kmax = 12
    prof = orj.LatencyProfile(np.full(kmax, 40, np.int64), 2 + np.arange(kmax, dtype=np.int64) // 3)
    gaps = rng.exponential(1.0, size=(S, n)) * rng.choice([5.0, 40.0, 400.0], size=(S, 1))
    arr = (np.cumsum(gaps, axis=1).astype(np.int64) + (1 << 40)).reshape(-1)
    dist = rng.integers(0, D, S * n).astype(np.int32)
    tb = np.concatenate([rng.choice(np.flatnonzero(counts[d]) + 1, 1) for d in dist]).astype(np.int16)
    off = np.arange(S + 1, dtype=np.int64) * n
    slo = rng.integers(200, 3000, S).astype(np.int64)
    tr = _trace(off, arr, dist, tb, slo)
    for G in (3, 16):
        pb0, log0, pb1, log1, pb2 = _both(store, prof, tr, G)
        assert (pb1 == pb0).all() and (pb2 == pb0).all() and (log1 == log0).all(), G
    assert pb0[:, 4].sum() > S  # scenarios actually batched


def test_size_guard_flags_short_num_arrivals():
    """The segmented replay sizes its scratch logs from the caller's
    num_arrivals: a value below arrival_offsets[S] must not write out of
    bounds -- the call does nothing and sets the size-error diagnostic."""
    import ctypes
    from paper_2209_00159_b200 import _abi
    tf, off, arr, dist, tb, slo = _family("gpt", 1, 3000)
    store = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
    prof = orj.LatencyProfile(tf.profile.a, tf.profile.w)
    tr = _trace(off, arr, dist, tb, slo)
    G, short = 4, len(arr) // 2
    need = orj.replay_seg_workspace_bytes(tr, G, True)
    ws = torch.zeros(need + 4096, dtype=torch.uint8, device="cuda")
    pb = torch.zeros((tr.num_buckets, 7), dtype=torch.int64, device="cuda")
    log = torch.zeros(len(arr) + len(slo), dtype=torch.int32, device="cuda")
    pol = _abi.ReplayPolicyC(0, None, None, None, None, 0.0)
    need_short = _abi.lib().orloj_replay_seg_workspace(tr.num_scenarios, short, G, 1)
    st = _abi.lib().orloj_replay_trace_seg(store.c(), prof.c(), tr.c(), ctypes.byref(pol), G, short, ws.data_ptr(),
                                           need_short, pb.data_ptr(), log.data_ptr(), None)
    assert st == 0
    torch.cuda.synchronize()
    assert orj.replay_seg_stats(ws)["size_error"] == 1
    assert int(pb.abs().sum()) == 0 and int(log.abs().sum()) == 0
    assert int(ws[need_short:].abs().sum()) == 0          # nothing written past the declared workspace
