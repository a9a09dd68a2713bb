"""GPU parity: the Alg. 1 replay policy (orloj_replay_trace_ex, objective
ALG1) vs oracle/alg1.py.

Follow mode (as for the E_k replay): the oracle replays the
GPU's popped-member masks, checks each one is in its tie set (same candidate
size, popped members inside Q_bs, no unpopped member of Q_bs with a higher
fp64 priority beyond the fp32 priority tolerance) and the per-scenario
counters must then agree bit for bit.  The hand-traced cases of
tests/test_oracle_alg1.py run on the GPU too."""
import numpy as np
import pytest

import gen
import _parity as par
from oracle import alg1

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2209_00159_b200 as orj  # noqa: E402
from paper_2209_00159_b200 import policy  # noqa: E402

T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()  # noqa: E731


def _gpu_alg1(counts, bin_ticks, a, w, b, off, arr, dist, tb, slo, buckets=None, nb=1):
    store = orj.HistogramStore.from_counts(counts, bin_ticks)
    prof = orj.LatencyProfile(a, w)
    tab = orj.PriorityTable(store, prof, len(a), b)
    thr = T(policy.alg1_size_thresholds(counts, a, w), np.int64)
    S = len(slo)
    bk = np.zeros(S, np.int32) if buckets is None else buckets
    tr = orj.Trace(T(off, np.int64), T(arr, np.int64), T(dist, np.int32), T(tb, np.int16), T(slo, np.int64),
                   T(bk, np.int32), nb)
    pb, log = orj.replay_trace(store, prof, tr, decision_log=True, objective="alg1", priority=tab,
                               size_thresholds=thr)
    torch.cuda.synchronize()
    return pb.cpu().numpy(), log.cpu().numpy()


def _hand():
    counts = np.array([[8, 0, 0, 0]], np.uint32)
    return counts, np.array([0, 0, 0], np.int64), np.array([10, 15, 22], np.int64)


@pytest.mark.parametrize("arr,tb,slo,counters,log", [
    ([0, 0], [1, 1], 100, [2, 2, 0, 0, 1, 15, 15], [0b11]),
    ([-94, 0, 0], [1, 1, 1], 100, [3, 3, 0, 0, 2, 25, 109], [0b1, 0b11]),
    ([0, 1, 6, 31], [4, 1, 1, 1], 49, [4, 3, 1, 0, 2, 55, 55], [0b1, 0b110]),
    ([-100, -94, -70, -70], [4, 1, 1, 1], 100, [4, 4, 0, 0, 2, 62, 62], [0b1, 0b111]),
])
def test_hand_traces(arr, tb, slo, counters, log):
    counts, a, w = _hand()
    n = len(arr)
    pb, lg = _gpu_alg1(counts, 1, a, w, 0.01, np.array([0, n]), np.array(arr), np.zeros(n), np.array(tb),
                       np.array([slo]))
    assert list(pb[0]) == counters
    assert list(lg[:len(log) + 1]) == log + [0]


@pytest.mark.parametrize("name", ["skipnet", "rdi", "gpt", "static"])
def test_follow_mode_parity(name):
    tf = gen.c5_trace_family(name)
    nb = len(gen.BUCKET_SLO_MULTS)
    gids = np.arange(nb, dtype=np.uint64)
    n = 1500
    arr, dist, tb = gen.trace_host(tf, gids, n)
    off = np.arange(nb + 1, dtype=np.int64) * n
    slo = np.array([tf.slo_of_bucket(b) for b in range(nb)], np.int64)
    b = 1.0 / tf.fam.mean_ticks()
    pb, lg = _gpu_alg1(tf.fam.counts, tf.fam.bin_ticks, tf.profile.a, tf.profile.w, b, off, arr, dist, tb, slo,
                       np.arange(nb, dtype=np.int32), nb)
    thr = alg1.size_thresholds(tf.fam.counts, tf.profile.a, tf.profile.w)
    ref = alg1.replay(tf.fam.counts, tf.profile.a, tf.profile.w, b, off, arr, dist, tb, slo, thr, follow_log=lg)
    assert (ref["ties"][:, 2] == -1).all(), ref["ties"]
    assert np.array_equal(ref["counters"], pb)  # one scenario per bucket
    # the popped sets differ from the oracle's own choice only at near-ties
    par.record("replay_ties", label=f"alg1/{name}", decisions=int(ref["ties"][:, 0].sum()),
               differing_choices=int(ref["ties"][:, 1].sum()), scenarios=nb)
    assert ref["ties"][:, 1].sum() <= 0.01 * ref["ties"][:, 0].sum() + 2
