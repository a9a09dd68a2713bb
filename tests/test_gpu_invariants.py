"""T2: invariants of the GPU outputs themselves, independent of the
oracle: P in [0, 1]; P_r(k+1) <= P_r(k) for a non-decreasing profile (A14:
log2F <= 0, RN addition and the integer lookup are monotone, so LG and
therefore P can only fall as the batch grows); E_k <= k; E_1 = P_1(1); point
masses give P in {0, 1} exactly."""
import numpy as np
import pytest

import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402


def _unpack(P, kmax):
    """packed [Q][kmax(kmax+1)/2] (index k(k-1)/2 + r) -> [Q][kmax][kmax] with NaN where r >= k"""
    Q = P.shape[0]
    out = np.full((Q, kmax, kmax), np.nan, np.float32)
    for k in range(1, kmax + 1):
        out[:, k - 1, :k] = P[:, k * (k - 1) // 2:k * (k + 1) // 2]
    return out


def _check(store, prof, qs, lens, kmax, point_mass=False):
    sc = orj.score_batches(store, prof, qs, want_P=True)
    e_only = orj.score_batches(store, prof, qs)["E"]
    torch.cuda.synchronize()
    P = _unpack(sc["P"].cpu().numpy(), kmax)
    K = np.minimum(lens, kmax)
    for E in (sc["E"].cpu().numpy(), e_only.cpu().numpy()):
        assert (E <= np.arange(1, kmax + 1)[None, :]).all()                       # E_k <= k
        nz = K > 0
        assert (E[nz, 0] == P[nz, 0, 0]).all()                                    # E_1 = P_1(1)
    for q in range(len(lens)):
        Pq = P[q, :K[q], :K[q]]
        v = Pq[~np.isnan(Pq)]
        assert ((v >= 0) & (v <= 1)).all()
        if point_mass:
            assert np.isin(v, [0.0, 1.0]).all()
        # P_r(k+1) <= P_r(k) for every member r < k, bit for bit
        for k in range(1, K[q]):
            assert (Pq[k, :k] <= Pq[k - 1, :k]).all(), (q, k)


def test_invariants_c2():
    c = gen.config2(Q=200)
    _check(wl.score_store(c), wl.profile(c.profile), wl.device_queues(c.queues), np.diff(c.queues.offsets), c.kmax)


def test_invariants_c3_rows():
    cfg = gen.config3(Q=64, n=256, kmax=64, T=128)
    store = wl.c3_store(cfg)
    _check(store, wl.profile(cfg.profile), wl.device_queues(cfg.queues), np.diff(cfg.queues.offsets), cfg.kmax)


def test_invariants_point_masses():
    c = gen.config4(Q=300)
    _check(wl.score_store(c), wl.profile(c.profile), wl.device_queues(c.queues), np.diff(c.queues.offsets), c.kmax,
           point_mass=True)


def test_determinism():
    """T5: reruns on the same inputs are byte-identical (pick, score with
    P, segmented replay with its log)."""
    c = gen.config2(Q=300)
    store, prof, qs = wl.score_store(c), wl.profile(c.profile), wl.device_queues(c.queues)
    runs = []
    for _ in range(2):
        bk, bE = orj.pick_batch(store, prof, qs)
        sc = orj.score_batches(store, prof, qs, want_P=True, want_EL=True)
        runs.append([bk.cpu().numpy(), bE.cpu().numpy()] + [sc[k].cpu().numpy() for k in ("E", "P", "EL")])
    for a, b in zip(*runs):
        assert a.tobytes() == b.tobytes()
    fam = wl.C5Family("rdi", local_ids=np.arange(24), n_arr=8000)
    logs = []
    for _ in range(2):
        pb, log = orj.replay_trace(fam.store, fam.profile, fam.trace, decision_log=True, segments=9)
        logs.append((pb.cpu().numpy().tobytes(), log.cpu().numpy().tobytes()))
    assert logs[0] == logs[1]
