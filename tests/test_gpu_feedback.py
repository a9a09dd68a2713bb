"""GPU parity of the long-term feedback loop (SURVEY §8(f) item 3,
PAPER.md:385-394, reading R15) against oracle/feedback.py.

* orloj_replay_trace_epoch: per-arrival outcomes, the carried worker time and
  the per-epoch counters equal the oracle's (follow mode) bit for bit;
* orloj_replay_feedback on a drifting trace (half the applications become
  1.5x slower half-way through): the oracle follows the GPU's per-epoch logs
  with its OWN store, rebuilt from its own window; counters and window counts
  bit-exact every epoch, the final store rows are RN32(log2 F) of the
  oracle's final F (F = 0 exactly where the GPU has -inf);
* one epoch with no refresh is the plain replay, bit for bit.
"""
import numpy as np
import pytest

import gen
import oracle
import _parity as par
from oracle import feedback as ofb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402

INT64_MIN = np.iinfo(np.int64).min


def _trace(off, arr, dist, tb, slo, bucket=None, nb=None):
    S = len(slo)
    bucket = np.arange(S) if bucket is None else bucket
    return orj.Trace(wl.t(off, np.int64), wl.t(arr, np.int64), wl.t(dist, np.int32), wl.t(tb, np.int16),
                     wl.t(slo, np.int64), wl.t(bucket, np.int32), S if nb is None else nb)


def _family(name, seeds, n):
    tf = gen.c5_trace_family(name)
    gids, bucket, slo = gen.c5_scenarios(tf, seeds)
    arr, dist, tb = gen.trace_host(tf, gids, n)
    off = np.arange(len(gids) + 1, dtype=np.int64) * n
    return tf, off, arr, dist, tb, slo


@pytest.mark.parametrize("fam", gen.C5_FAMILIES)
def test_epochs_outcomes_and_worker_carry(fam):
    tf, off, arr, dist, tb, slo = _family(fam, 2, 6000)
    E = 4
    store = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
    prof = orj.LatencyProfile(tf.profile.a, tf.profile.w)
    tr = _trace(off, arr, dist, tb, slo)
    S, N = len(slo), len(arr)
    wf = torch.full((S,), INT64_MIN, dtype=torch.int64, device="cuda")
    oc = torch.zeros(N, dtype=torch.uint8, device="cuda")
    F = oracle.cdf(tf.fam.counts)
    t_or = np.full(S, INT64_MIN, np.int64)
    for e in range(E):
        pb, log = orj.replay_epoch(store, prof, tr, e, E, worker_free=wf, outcome=oc, decision_log=True)
        torch.cuda.synchronize()
        idx, sub_off = ofb.epoch_index(off, e, E)
        ref = oracle.replay(F, tf.profile.a, tf.profile.w, sub_off, arr[idx], dist[idx], tb[idx], slo,
                            follow_log=ofb.epoch_log_view(log.cpu().numpy(), off, e, E), t_start=t_or,
                            want_outcome=True)
        par.check_replay_follow(ref, pb.cpu().numpy(), f"epoch{e}/{fam}")
        t_or = ref["t_end"]
        assert (wf.cpu().numpy() == t_or).all(), e
        assert (oc.cpu().numpy()[idx] == ref["outcome"]).all(), e
    assert set(np.unique(oc.cpu().numpy()).tolist()) <= {1, 2, 3}


def test_one_epoch_no_refresh_is_plain_replay():
    tf, off, arr, dist, tb, slo = _family("skipnet", 2, 8000)
    prof = orj.LatencyProfile(tf.profile.a, tf.profile.w)
    tr = _trace(off, arr, dist, tb, slo)
    st0 = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
    plain, plog = orj.replay_trace(st0, prof, tr, decision_log=True)
    st1 = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
    before = st1.log2_cdf.clone()
    out = orj.replay_feedback(st1, prof, tr, num_epochs=1, window_epochs=1, min_samples=1 << 31,
                              decision_logs=True)
    torch.cuda.synchronize()
    assert torch.equal(out["per_epoch"][0], plain)
    assert torch.equal(out["logs"][0], plog)
    assert torch.equal(st1.log2_cdf, before)                   # no row reached min_samples
    # the window holds every completed request (no sample mask)
    w = out["window"].cpu().numpy().astype(np.int64)
    c = plain.cpu().numpy()
    assert w.sum() == c[:, 1].sum() + c[:, 3].sum()


@pytest.mark.parametrize("fam", ["skipnet", "gpt", "rdi"])
def test_feedback_loop_vs_oracle(fam):
    tf = gen.c5_trace_family(fam)
    gids, bucket, slo = gen.c5_scenarios(tf, 2)
    n, E, W, m = 12_000, 6, 2, 200
    arr, dist, tb, tfd = gen.drift_trace_host(tf, gids, n, E, E // 2)
    off = np.arange(len(gids) + 1, dtype=np.int64) * n
    mask = gen.sample_mask(gen.SEED_BASE + 40, len(arr), 0.25)
    prof = orj.LatencyProfile(tf.profile.a, tf.profile.w)
    tr = _trace(off, arr, dist, tb, slo)
    store = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)      # prior: the pre-drift profile
    out = orj.replay_feedback(store, prof, tr, num_epochs=E, window_epochs=W, min_samples=m,
                              sample_mask=wl.t(mask, np.uint8), decision_logs=True)
    torch.cuda.synchronize()
    logs = out["logs"].cpu().numpy()
    ref = ofb.replay_feedback(tf.fam.counts, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo, E, W, m,
                              sample_mask=mask, follow_logs=logs)
    got = out["per_epoch"].cpu().numpy()
    for e in range(E):
        par.check_replay_follow({"ties": ref["ties"][e], "counters": ref["counters"][e]}, got[e],
                                f"feedback/{fam}/epoch{e}")
    assert (out["window"].cpu().numpy().astype(np.int64) == ref["window"]).all()
    assert ref["refreshed"].any(), "no row was ever refreshed: the loop was not exercised"
    # the final store: the oracle's final F read through the store format
    L = store.log2_cdf.cpu().numpy()
    Fo = ref["F"]
    assert (np.isneginf(L) == (Fo == 0)).all()
    fin = Fo > 0
    assert np.abs(np.exp2(L[fin].astype(np.float64)) - Fo[fin]).max() <= 1e-6
    assert (L[:, -1] == 0).all()
    # the drifted applications' rows moved towards the drifted histograms
    slow = np.arange(tf.fam.D // 2)
    mean_bin = lambda Fr: (1.0 - Fr[:, :-1]).sum(1) + 1.0          # noqa: E731
    prior = oracle.cdf(tf.fam.counts)
    assert (mean_bin(Fo[slow]) > mean_bin(prior[slow])).all()
