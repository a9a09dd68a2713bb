"""GPU parity of the replay policy variants (orloj_replay_trace_ex;
SURVEY §8(f) item 1): finish-rate objective E_k / E[L_{B_k}] and the Alg. 1
expected-latency drop, against the oracle in follow mode (decisions within the
tie set, integer counters bit-exact) and on hand-derived golden cases."""
import numpy as np
import pytest

import gen
import oracle
import _parity as par

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import _policy_cases  # noqa: E402

import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402
from paper_2209_00159_b200 import policy  # noqa: E402


def _run(store, prof, off, arr, dist, tb, slo, objective, thr):
    S = len(slo)
    tr = orj.Trace(wl.t(off, np.int64), wl.t(arr, np.int64), wl.t(dist, np.int32), wl.t(tb, np.int16),
                   wl.t(slo, np.int64), wl.t(np.arange(S), np.int32), S)
    pb, log = orj.replay_trace(store, prof, tr, decision_log=True, objective=objective,
                               drop_threshold=None if thr is None else wl.t(thr, np.int64))
    torch.cuda.synchronize()
    return pb.cpu().numpy(), log.cpu().numpy()


@pytest.mark.parametrize("case", _policy_cases.load(), ids=lambda c: c["name"])
def test_policy_golden_gpu(case):
    x = _policy_cases.arrays(case)
    store = orj.HistogramStore.from_counts(x["counts"], 1)
    prof = orj.LatencyProfile(x["a"], x["w"])
    for key, exp in case["expect"].items():
        objective, drop = key.split("/")
        thr = policy.expected_latency_thresholds(x["counts"], x["a"], x["w"]) if drop == "expected_latency" else None
        pb, _ = _run(store, prof, x["off"], x["arrival"], x["dist"], x["tb"], x["slo"], objective, thr)
        assert dict(zip(orj.COUNTER_FIELDS, pb[0].tolist())) == exp, key


@pytest.mark.parametrize("fam", gen.C5_FAMILIES)
@pytest.mark.parametrize("objective,drop", [("finish_rate", "hopeless"), ("expected_finish", "expected_latency"),
                                            ("finish_rate", "expected_latency")])
def test_policy_follow_mode(fam, objective, drop):
    tf = gen.c5_trace_family(fam)
    gids, bucket, slo = gen.c5_scenarios(tf, 4)
    n = 8000
    arr, dist, tb = gen.trace_host(tf, gids, n)
    off = np.arange(len(gids) + 1, dtype=np.int64) * n
    store = orj.HistogramStore.from_counts(tf.fam.counts, tf.fam.bin_ticks)
    prof = orj.LatencyProfile(tf.profile.a, tf.profile.w)
    thr = policy.expected_latency_thresholds(tf.fam.counts, tf.profile.a, tf.profile.w) \
        if drop == "expected_latency" else None
    pb, log = _run(store, prof, off, arr, dist, tb, slo, objective, thr)
    ref = oracle.replay(oracle.cdf(tf.fam.counts), tf.profile.a, tf.profile.w, off, arr, dist, tb, slo,
                        follow_log=log, objective=objective, drop=drop, counts=tf.fam.counts)
    free = oracle.replay(oracle.cdf(tf.fam.counts), tf.profile.a, tf.profile.w, off, arr, dist, tb, slo,
                         objective=objective, drop=drop, counts=tf.fam.counts)
    # the rate objective's tie band is relative (1e-4 rate_max): allow 1e-4 of the decisions
    par.check_replay_follow(ref, pb, f"policy/{fam}/{objective}/{drop}",
                            tie_rate=1e-4 if objective == "finish_rate" else 1e-5, free=free)
    # explicit hopeless thresholds reproduce the built-in rule exactly
    if drop == "hopeless":
        pb2, log2 = _run(store, prof, off, arr, dist, tb, slo, objective,
                         policy.hopeless_thresholds(tf.fam.counts, tf.profile.a, tf.profile.w))
        assert (pb2 == pb).all() and (log2 == log).all()
