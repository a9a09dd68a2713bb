"""GPU parity at the full C5 size (BASELINE.json config 5), in the launch
configuration bench.py times: each family's 2,048 scenarios x 100,000 arrivals
replayed by the segmented kernel (8 segments per scenario, bench.py's "auto"
at one GPU).  The oracle cannot replay 205 M arrivals, so it follows the GPU's
decision log on sampled scenarios (the first and last scenario and random ones
over all SLO buckets): decisions within its tie sets, counters bit-exact
(SURVEY §8(c) O2).  The per-bucket table the bench reads must equal the sum of
the per-scenario counters."""
import numpy as np
import pytest

import gen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402

SEGMENTS = 8


@pytest.mark.parametrize("fam", gen.C5_FAMILIES)
def test_c5_full_size_sampled(fam):
    f = wl.C5Family(fam)
    S, n = f.num_scenarios, f.n_arr
    assert S == 2048 and n == 100_000
    per_scen = orj.Trace(f.trace.offsets, f.trace.arrival, f.trace.dist, f.trace.true_bin, f.trace.slo,
                         torch.arange(S, dtype=torch.int32, device="cuda"), S)
    pb, log = orj.replay_trace(f.store, f.profile, per_scen, decision_log=True, segments=SEGMENTS)
    table, _ = orj.replay_trace(f.store, f.profile, f.trace, segments=SEGMENTS)   # the bench's call
    torch.cuda.synchronize()
    pb = pb.cpu().numpy()
    tab = table.cpu().numpy()
    expect = np.zeros_like(tab)
    np.add.at(expect, f.bucket_np, pb)   # every counter (span included) is summed per bucket
    assert (tab == expect).all()
    assert (pb[:, 1] + pb[:, 2] + pb[:, 3] == pb[:, 0]).all() and (pb[:, 0] == n).all()

    rng = np.random.default_rng(20220905)
    sample = np.unique(np.concatenate([[0, S - 1], rng.choice(S, 4, replace=False)]))
    F = oracle.cdf(f.tf.fam.counts)
    for s in sample:
        lo = s * n
        arr = f.trace.arrival[lo:lo + n].cpu().numpy()
        dist = f.trace.dist[lo:lo + n].cpu().numpy()
        tb = f.trace.true_bin[lo:lo + n].cpu().numpy()
        lg = log[lo + s:lo + s + n + 1].cpu().numpy()
        ref = oracle.replay(F, f.tf.profile.a, f.tf.profile.w, np.array([0, n], np.int64), arr, dist, tb,
                            f.slo_np[s:s + 1], follow_log=lg)
        assert (ref["ties"][:, 2] == -1).all(), (fam, s)
        assert (ref["counters"][0] == pb[s]).all(), (fam, s, ref["counters"][0], pb[s])
