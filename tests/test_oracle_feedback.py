"""Pins of oracle/feedback.py and of the replay's per-arrival outcomes and
carried worker time (reading R15),
against hand-traced cases, the window arithmetic and the SPEC's drift
example, independent of the loop's own code."""
import numpy as np

import gen
import oracle
from oracle import feedback as fb


def _point_store(B, bins):
    counts = np.zeros((len(bins), B), np.uint32)
    for d, i in enumerate(bins):
        counts[d, i - 1] = 1 << 30
    return counts


def test_outcomes_agree_with_counters():
    """Every arrival gets exactly one outcome, and their counts per scenario are
    the finished / late / dropped counters."""
    tf = gen.c5_trace_family("rdi")
    gids, bucket, slo = gen.c5_scenarios(tf, 2)
    n = 3000
    arr, dist, tb = gen.trace_host(tf, gids, n)
    off = np.arange(len(gids) + 1, dtype=np.int64) * n
    r = oracle.replay(oracle.cdf(tf.fam.counts), tf.profile.a, tf.profile.w, off, arr, dist, tb, slo,
                      want_outcome=True)
    oc = r["outcome"].reshape(len(gids), n)
    assert set(np.unique(oc)) <= {1, 2, 3}
    for code, col in ((1, 1), (3, 2), (2, 3)):
        assert ((oc == code).sum(1) == r["counters"][:, col]).all()
    assert (oc == 3).any() and (oc == 2).any()


def test_spec_example_outcomes():
    """SPEC S:430 (4 requests at t = 0, true times 10, 10, 100, 100 ms, SLO 150,
    dur = k max): three finish, one is dropped -- the outcome codes say which."""
    B = 100
    counts = np.zeros((2, B), np.uint32)
    counts[0, 9] = counts[1, 99] = 1
    a, w = np.zeros(4, np.int64), np.arange(1, 5, dtype=np.int64)
    arr = np.zeros(4, np.int64)
    dist = np.array([0, 0, 1, 1], np.int32)
    tb = np.array([10, 10, 100, 100], np.int16)
    r = oracle.replay(oracle.cdf(counts), a, w, np.array([0, 4]), arr, dist, tb, np.array([150]),
                      want_outcome=True)
    assert r["counters"][0].tolist()[:4] == [4, 3, 1, 0]
    assert sorted(r["outcome"].tolist()) == [1, 1, 1, 3]


def test_epoch_barrier_and_worker_carry_hand_case():
    """Hand trace: 3 requests at t = 0 (point mass in bin 2, Delta = 1 tick,
    a = 0, w_k = k, SLO 100), two epochs: epoch 0 = request 0 alone
    (dur 2, ends at 2); epoch 1 = requests 1, 2, admitted when the worker is
    free at 2, batched (E_2 = 2 > E_1 = 1), dur 2 * 2 = 4, ends at 6."""
    counts = _point_store(4, [2])
    a, w = np.zeros(3, np.int64), np.arange(1, 4, dtype=np.int64)
    r = fb.replay_feedback(counts, a, w, np.array([0, 3]), np.zeros(3, np.int64), np.zeros(3, np.int32),
                           np.full(3, 2, np.int16), np.array([100]), num_epochs=2, window_epochs=1,
                           min_samples=1 << 30)
    c = r["counters"]
    assert c[0, 0].tolist() == [1, 1, 0, 0, 1, 2, 2]
    assert c[1, 0].tolist() == [2, 2, 0, 0, 1, 4, 6]
    assert r["outcome"].tolist() == [1, 1, 1]
    # one epoch: all three in one window, batched together (dur 3 * 2 = 6)
    r1 = fb.replay_feedback(counts, a, w, np.array([0, 3]), np.zeros(3, np.int64), np.zeros(3, np.int32),
                            np.full(3, 2, np.int16), np.array([100]), num_epochs=1, window_epochs=1,
                            min_samples=1 << 30)
    assert r1["counters"][0, 0].tolist() == [3, 3, 0, 0, 1, 6, 6]
    # a worker busy until 50 (t_start) delays everything: ends at 50 + 6
    r2 = oracle.replay(oracle.cdf(counts), a, w, np.array([0, 3]), np.zeros(3, np.int64), np.zeros(3, np.int32),
                       np.full(3, 2, np.int16), np.array([100]), t_start=np.array([50]))
    assert r2["t_end"].tolist() == [56] and r2["counters"][0, 1] == 3


def test_one_epoch_is_the_plain_replay():
    tf = gen.c5_trace_family("skipnet")
    gids, _, slo = gen.c5_scenarios(tf, 1)
    n = 2000
    arr, dist, tb = gen.trace_host(tf, gids, n)
    off = np.arange(len(gids) + 1, dtype=np.int64) * n
    plain = oracle.replay(oracle.cdf(tf.fam.counts), tf.profile.a, tf.profile.w, off, arr, dist, tb, slo)
    r = fb.replay_feedback(tf.fam.counts, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo, 1, 1, 1 << 30)
    assert (r["counters"][0] == plain["counters"]).all()


def test_window_reset_arithmetic():
    """W = 2 over E = 5 epochs: the last refresh uses the window of epoch 4
    alone (reset after epochs 1 and 3), i.e. the histogram of epoch 4's
    sampled completed requests, computed here straight from the outcomes."""
    tf = gen.c5_trace_family("gpt")
    gids, _, slo = gen.c5_scenarios(tf, 1)
    n, E = 2500, 5
    arr, dist, tb = gen.trace_host(tf, gids, n)
    off = np.arange(len(gids) + 1, dtype=np.int64) * n
    mask = gen.sample_mask(7, len(arr), 0.25)
    r = fb.replay_feedback(tf.fam.counts, tf.profile.a, tf.profile.w, off, arr, dist, tb, slo, E, 2, 50,
                           sample_mask=mask)
    idx, _ = fb.epoch_index(off, E - 1, E)
    sel = idx[np.isin(r["outcome"][idx], (1, 2)) & (mask[idx] == 1)]
    expect = np.zeros_like(r["window"])
    np.add.at(expect, (dist[sel], tb[sel].astype(np.int64) - 1), 1)
    assert (r["window"] == expect).all() and expect.sum() > 0
    # every epoch's rows with >= 50 window samples were rebuilt; the final F rows are the window's CDF
    rows = r["refreshed"][-1]
    assert rows.any()
    for d in np.nonzero(rows)[0]:
        assert np.array_equal(r["F"][d], np.cumsum(expect[d]) / expect[d].sum())


def test_drift_moves_the_mass():
    """all mass moves from 10 to 100 ms: after one full window and
    a refresh the old mode's mass is gone.  Prior: point mass in bin 1; every
    request truly takes bin 10; W = 1, min_samples = 1."""
    B = 12
    counts = _point_store(B, [1])
    a, w = np.zeros(4, np.int64), np.arange(1, 5, dtype=np.int64)
    n = 40
    arr = np.arange(n, dtype=np.int64) * 100
    r = fb.replay_feedback(counts, a, w, np.array([0, n]), arr, np.zeros(n, np.int32), np.full(n, 10, np.int16),
                           np.array([10 ** 6]), num_epochs=2, window_epochs=1, min_samples=1)
    F = r["F"][0]
    assert (F[:9] == 0).all() and (F[9:] == 1).all()
    assert r["window"][0].tolist() == [0] * 9 + [20, 0, 0]
