"""GPU parity at the full C5 size (BASELINE.json config 5), in the launch
configuration bench.py times: each family's 2,048 scenarios x 100,000 arrivals
replayed by the segmented kernel (8 segments per scenario, bench.py's "auto"
at one GPU).  The oracle follows the GPU's decision log on every scenario (one
OpenMP call per family, a few seconds on the host cores): decisions within
its tie sets, counters bit-exact, the number of documented ties reported and
bounded; its free run must equal the GPU run on every
scenario without a tie.  The per-bucket table the bench reads must equal the
sum of the per-scenario counters."""
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

SEGMENTS = 8


@pytest.mark.parametrize("fam", gen.C5_FAMILIES)
def test_c5_full_size_every_scenario(fam):
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

    # the oracle follows EVERY scenario's log (one OpenMP call over 2,048
    # scenarios), then replays them free: tie-free scenarios must be identical
    F = oracle.cdf(f.tf.fam.counts)
    arr = f.trace.arrival.cpu().numpy()
    dist = f.trace.dist.cpu().numpy()
    tb = f.trace.true_bin.cpu().numpy()
    lg = log.cpu().numpy()
    ref = oracle.replay(F, f.tf.profile.a, f.tf.profile.w, f.offsets_np, arr, dist, tb, f.slo_np, follow_log=lg)
    free = oracle.replay(F, f.tf.profile.a, f.tf.profile.w, f.offsets_np, arr, dist, tb, f.slo_np)
    st = par.check_replay_follow(ref, pb, f"C5-full/{fam}", free=free)
    assert st["decisions"] == int(pb[:, 4].sum())
