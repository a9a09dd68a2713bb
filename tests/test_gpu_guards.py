"""Out-of-bounds write guards (T4 without compute-sanitizer, which this GPU pool
closed): every output a C-ABI call writes is a view into a larger buffer whose
head and tail hold a byte pattern; after the call the pattern must be intact
and the view must equal an unguarded run of the same call.  Shapes are small,
odd and ragged so that every kernel's tail handling runs (TMA ring and
shared-memory store score paths, the short-queue kernel, priorities with the
vector and strided member maps, both PopBatch paths, the plain and segmented
replays with decision logs, the model-variant kernels)."""
import numpy as np
import pytest

import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402

GUARD = 4096          # bytes on each side (keeps the 256-byte alignment of workspaces)
PATTERN = 0xA5


class Guarded:
    """A device view of `shape` x `dtype` with GUARD pattern bytes on both sides."""

    def __init__(self, shape, dtype, fill=None):
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        self.raw = torch.full((GUARD + n + GUARD,), PATTERN, dtype=torch.uint8, device="cuda")
        self.n = n
        self.view = self.raw[GUARD:GUARD + n].view(dtype).view(*shape)
        if fill is not None:
            self.view.fill_(fill)

    def intact(self) -> bool:
        torch.cuda.synchronize()
        return bool((self.raw[:GUARD] == PATTERN).all()) and bool((self.raw[GUARD + self.n:] == PATTERN).all())


def _same(a, b):
    return torch.equal(a.contiguous().view(torch.uint8), b.contiguous().view(torch.uint8))


@pytest.mark.parametrize("which", ["C1", "C2", "C3small", "C4small"])
def test_score_and_pick_guards(which):
    if which == "C1":
        c = gen.config1()
        st = orj.HistogramStore.from_counts(c.fam.counts, c.fam.bin_ticks)
    elif which == "C2":
        c = gen.config2(Q=37)
        st = orj.HistogramStore.from_counts(c.fam.counts, c.fam.bin_ticks)
    elif which == "C3small":
        c = gen.config3(Q=19, n=80, kmax=64, T=64)
        st = wl.c3_store(c)
    else:
        c = gen.config4(Q=45)
        st = orj.HistogramStore.from_counts(c.fam.counts, c.fam.bin_ticks)
    pr = wl.profile(c.profile)
    q = wl.device_queues(c.queues)
    Q, K = c.queues.Q, pr.kmax
    bk, bE = Guarded((Q,), torch.int32), Guarded((Q,), torch.float32)
    orj.pick_batch(st, pr, q, bk.view, bE.view)
    rk, rE = orj.pick_batch(st, pr, q)
    assert bk.intact() and bE.intact()
    assert _same(bk.view, rk) and _same(bE.view, rE)
    for want_P, want_EL in ((False, False), (True, True)):
        E = Guarded((Q, K), torch.float32)
        out = {"E": E.view}
        P = EL = None
        if want_P:
            P = Guarded((Q, K * (K + 1) // 2), torch.float32, fill=0.0)
            out["P"] = P.view
        if want_EL:
            EL = Guarded((Q, K), torch.float32)
            out["EL"] = EL.view
        orj.score_batches(st, pr, q, want_P=want_P, want_EL=want_EL, out=out)
        ref = orj.score_batches(st, pr, q, want_P=want_P, want_EL=want_EL)
        for g, name in ((E, "E"), (P, "P"), (EL, "EL")):
            if g is not None:
                assert g.intact(), name
                assert _same(g.view, ref[name]), name


def test_priority_and_pop_guards():
    cp = gen.config_priority(Q=13, n=256)
    cp.queues.offsets[6:] -= 3   # a short queue and unaligned chunks next to full ones
    st = orj.HistogramStore.from_counts(cp.fam.counts, cp.fam.bin_ticks)
    q = wl.device_queues(cp.queues)
    N, Q = int(cp.queues.offsets[-1] - cp.queues.offsets[0]), cp.queues.Q
    for b in (1.0 / cp.fam.mean_ticks(), 50.0 / cp.fam.mean_ticks()):
        tab = orj.PriorityTable(st, wl.profile(cp.profile), 32, b)
        lp = Guarded((32, N), torch.float32)
        tab.scores(q, out=lp.view)
        ref = tab.scores(q)
        assert lp.intact() and _same(lp.view, ref)
        for bs, src in ((32, ref), (5, torch.zeros_like(ref))):   # fast path, general path (all tied)
            size = torch.full((Q,), bs, dtype=torch.int32, device="cuda")
            sel = Guarded((Q, 32), torch.int32)
            tab.pop(q, src, size, out=sel.view)
            assert sel.intact() and _same(sel.view, tab.pop(q, src, size))


@pytest.mark.parametrize("segments", [1, 7])
def test_replay_guards(segments):
    f = wl.C5Family("rdi", local_ids=np.arange(11), n_arr=3001)
    S, N, nb = f.trace.num_scenarios, f.trace.num_arrivals, f.trace.num_buckets
    pb = Guarded((nb, 7), torch.int64, fill=0)
    log = Guarded((N + S,), torch.int32, fill=0)
    ws = None
    if segments > 1:
        ws = Guarded((orj.replay_seg_workspace_bytes(f.trace, segments, True),), torch.uint8)
    orj.replay_trace(f.store, f.profile, f.trace, per_bucket=pb.view, decision_log=log.view, segments=segments,
                     workspace=None if ws is None else ws.view)
    rpb, rlog = orj.replay_trace(f.store, f.profile, f.trace, decision_log=True)
    assert pb.intact() and log.intact() and (ws is None or ws.intact())
    assert torch.equal(pb.view, rpb) and torch.equal(log.view, rlog)


def test_model_variant_guards():
    c2 = gen.config2(Q=21)
    st2 = orj.HistogramStore.from_counts(c2.fam.counts, c2.fam.bin_ticks)
    q2 = wl.device_queues(c2.queues)
    m = np.arange(c2.fam.B + 1, dtype=np.int64)
    eq3 = c2.profile.a[:, None] + c2.profile.w[:, None] * m[None, :]
    for interp in (False, True):
        for steps in (None, ([0, 300], [1.0, 1.5])):
            model = orj.ScoreModel(eq3, interpolate=interp, steps=steps)
            ref = model.score(st2, q2)
            out = {k: Guarded(tuple(v.shape), v.dtype) for k, v in ref.items() if isinstance(v, torch.Tensor)}
            model.score(st2, q2, out={k: g.view for k, g in out.items()})
            for k, g in out.items():
                assert g.intact(), k
                assert _same(g.view, ref[k]), k
