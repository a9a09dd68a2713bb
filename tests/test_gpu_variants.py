"""GPU parity: scoring-model variants (orloj_score_model_batches, SURVEY
§8(f) item 4) vs oracle/variants.py.  Tolerances as the main scorer
 scaled by the step weights: |E_k| within 2e-5 k sum(dc) (the
uniform-bin product adds k fp32 factors, each from ex2.approx), k* exact
except documented ties (the rule of SURVEY §8(c))."""
import numpy as np
import pytest

import gen
from oracle import variants as va

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402

KMAX = 16


def _case(seed):
    fam = gen.skipnet_family(seed)
    prof = gen.eq3_half(fam, KMAX)
    rng = np.random.default_rng(seed + 1)
    lengths = rng.integers(0, 22, 20)
    lengths[:4] = (0, 1, KMAX, 21)
    q = gen.snapshot_queues(seed, lengths, fam.p99_ticks(), D=fam.D)
    return fam, prof, q


def _tables(fam, prof):
    B = fam.B
    m = np.arange(B + 1, dtype=np.int64)
    eq3 = prof.a[:, None] + prof.w[:, None] * m[None, :]
    # log-spaced grid: position m at a_k + w_k B (2^{m/B * 4} - 1) / 15, non-decreasing, same horizon
    logm = np.round(B * (2.0 ** (4.0 * m / B) - 1.0) / 15.0).astype(np.int64)
    logt = prof.a[:, None] + prof.w[:, None] * logm[None, :]
    return {"eq3": eq3, "log": logt}


def _check(E_g, bk_g, E_o, bk_o, lens, tol_k):
    K = np.minimum(lens, KMAX)
    k = np.arange(1, KMAX + 1)
    err = np.abs(E_g.astype(np.float64) - E_o)
    assert (err <= tol_k * k[None, :] + 1e-7).all(), float(err.max())
    assert ((bk_g == 0) == (K == 0)).all()
    for q in np.nonzero(bk_g != bk_o)[0]:
        kg, ko = int(bk_g[q]), int(bk_o[q])
        eg, eo = abs(E_g[q, kg - 1] - E_o[q, kg - 1]), abs(E_g[q, ko - 1] - E_o[q, ko - 1])
        assert E_o[q, ko - 1] - E_o[q, kg - 1] <= eg + eo + 1e-12


@pytest.mark.parametrize("table", ["eq3", "log"])
@pytest.mark.parametrize("interp", [False, True])
@pytest.mark.parametrize("steps", [None, ([-200, 0, 900], [0.25, 1.0, 1.5])])
def test_model_vs_oracle(table, interp, steps):
    fam, prof, q = _case(gen.SEED_BASE + 950)
    dur = _tables(fam, prof)[table]
    store = orj.HistogramStore.from_counts(fam.counts, fam.bin_ticks)
    qs = wl.device_queues(q)
    model = orj.ScoreModel(dur, interpolate=interp, steps=steps)
    out = model.score(store, qs)
    torch.cuda.synchronize()
    so, sc = (steps if steps else ((0,), (1.0,)))
    E_o, bk_o = va.score(fam.counts, dur, q.offsets, q.deadline, q.dist, q.now, interp, so, sc)
    _check(out["E"].cpu().numpy(), out["best_k"].cpu().numpy(), E_o, bk_o, np.diff(q.offsets),
           2e-5 * float(sc[-1]))
    bE = out["best_E"].cpu().numpy()
    bk = out["best_k"].cpu().numpy()
    Eg = out["E"].cpu().numpy()
    nz = bk > 0
    assert (bE[nz] == Eg[nz, bk[nz] - 1]).all() and (bE[~nz] == 0).all()


def test_eq3_edge_unit_step_matches_main_scorer():
    """Same model as orloj_score_batches: the two kernels agree within the E tolerance."""
    fam, prof, q = _case(gen.SEED_BASE + 951)
    store = orj.HistogramStore.from_counts(fam.counts, fam.bin_ticks)
    qs = wl.device_queues(q)
    p = orj.LatencyProfile(prof.a, prof.w)
    main = orj.score_batches(store, p, qs)["E"]
    var = orj.ScoreModel.eq3(p, fam.B).score(store, qs)["E"]
    torch.cuda.synchronize()
    k = torch.arange(1, KMAX + 1, device="cuda")
    assert ((main - var).abs() <= 1e-5 * k).all()
    # the edge kernel on an arithmetic-grid table is the short-queue scorer's
    # arithmetic step for step (same adds, lookup constants, ex2, butterfly)
    assert torch.equal(main, var)


def test_model_without_plan_equals_planned():
    """orloj_score_model_batches with plan = NULL (row analysis on every call)
    gives the planned call's results bit for bit, for a grid table and for a
    table with a non-grid row (binary search), one and three steps."""
    import ctypes
    from paper_2209_00159_b200 import _abi
    fam, prof, q = _case(gen.SEED_BASE + 953)
    store = orj.HistogramStore.from_counts(fam.counts, fam.bin_ticks)
    qs = wl.device_queues(q)
    t = _tables(fam, prof)
    mixed = t["eq3"].copy()
    mixed[5] = t["log"][5]
    for dur in (t["eq3"], mixed):
        for steps in (None, ([-200, 0, 900], [0.25, 1.0, 1.5])):
            model = orj.ScoreModel(dur, steps=steps)
            planned = model.score(store, qs)
            c = model.c()
            c._obj.plan = None
            E = torch.empty_like(planned["E"])
            bk = torch.empty_like(planned["best_k"])
            bE = torch.empty_like(planned["best_E"])
            _abi.check(_abi.lib().orloj_score_model_batches(store.c(), qs.c(), c, E.data_ptr(), bk.data_ptr(),
                                                            bE.data_ptr(), torch.cuda.current_stream().cuda_stream))
            torch.cuda.synchronize()
            assert torch.equal(E, planned["E"]) and torch.equal(bk, planned["best_k"])


def test_invalid_models():
    fam, prof, q = _case(gen.SEED_BASE + 952)
    store = orj.HistogramStore.from_counts(fam.counts, fam.bin_ticks)
    qs = wl.device_queues(q)
    dur = _tables(fam, prof)["eq3"]
    with pytest.raises(orj.OrlojError):
        orj.ScoreModel(dur[:, ::-1])  # decreasing in m
    with pytest.raises(orj.OrlojError):
        orj.ScoreModel(np.tile(dur[:1], (33, 1)))  # kmax > 32
    with pytest.raises(orj.OrlojError):
        orj.ScoreModel(dur, steps=([0, 0], [1.0, 2.0])).score(store, qs)
    with pytest.raises(orj.OrlojError):
        orj.ScoreModel(dur[:, :33]).score(store, qs)  # table B != store B
