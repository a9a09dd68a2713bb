"""GPU parity: Eq. 1-2 priority scores and PopBatch (orloj_priority_table /
orloj_priority_scores / orloj_pop_batch) vs oracle/priority.py.

Tolerance on log p (R10-R12): the CUDA path reads the store,
whose data format is log2 F rounded to fp32 (include/orloj.h), and writes
fp32 log p.  The oracle reads the same format (oracle.priority
store_fp32=True: counts -> fp64 log2 F -> fp32, its own arithmetic).  The
tables are fp64 (error < 1e-9 after the bin-mass cancellation G_i - G_{i-1});
per element the full-bin term C[i*] - b sigma - log E[L] is formed in fp64 and
rounded once to fp32 (2^-24 relative), the partial-bin term is fp32 (its
log(h/b) - log E[L] rounded once, 1 - e^{-bx} by expm1f, <= 2 ulp), and the
log-add-exp (log1pf(exp(d)) in [0, ln 2], abs error < 2^-22) plus the final
add (2^-24 relative): |d log p| <= 1e-6 + 2^-22 |log p| (each term's relative
error enters with its softmax weight, so never more than the larger term's
share).  Against the exact-count model (Eq. 2 on the real histograms) the
store format adds at most oracle.priority.store_rounding_log_priority_bound
(first-order propagation of the one RN rounding of log2 F, pinned on CPU in
tests/test_oracle_priority.py); the GPU test asserts the sum of the two and
reports the elements where that bound is infinite (near-empty bins).
-inf (p = 0: no outcome of L_bs fits before the deadline) must match exactly.
PopBatch is integer work: bit-exact against the oracle on the same fp32
scores (seeded inputs, not GPU outputs).
"""
import numpy as np
import pytest

import gen
from oracle import priority as pr

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2209_00159_b200 as orj  # noqa: E402
import workloads as wl  # noqa: E402

S = 32


def _tol(ref):
    return 1e-6 + 2.0 ** -22 * np.abs(ref)


def _case(name, seed, Q=96):
    fam = {"skipnet": gen.skipnet_family, "rdi": gen.rdi_family, "gpt": gen.gpt_family}[name](seed)
    prof = gen.eq3_half(fam, S)
    rng = np.random.default_rng(seed + 7)
    lengths = rng.integers(0, 300, Q)
    lengths[:3] = (0, 1, 256)
    q = gen.snapshot_queues(seed, lengths, fam.p99_ticks(), D=fam.D)
    # a few queues observed after their deadlines (negative slack)
    q.now[4:8] += 3 * fam.p99_ticks()
    return fam, prof, q


def _gpu_scores(fam, prof, q, b, weights=None):
    store = orj.HistogramStore.from_counts(fam.counts, fam.bin_ticks)
    p = orj.LatencyProfile(prof.a, prof.w)
    wt = None if weights is None else torch.tensor(weights, dtype=torch.float32, device="cuda")
    tab = orj.PriorityTable(store, p, S, b, weights=wt)
    qs = wl.device_queues(q)
    lp = tab.scores(qs)
    torch.cuda.synchronize()
    return tab, qs, lp


@pytest.mark.parametrize("name", ["skipnet", "rdi", "gpt"])
@pytest.mark.parametrize("b_scale", [0.05, 1.0, 20.0])
def test_scores_vs_oracle(name, b_scale):
    fam, prof, q = _case(name, gen.SEED_BASE + 910)
    b = b_scale / fam.mean_ticks()  # anticipated delay ~ mean latency / b_scale
    weights = None if b_scale != 1.0 else np.linspace(0.5, 2.0, fam.D)
    _, _, lp = _gpu_scores(fam, prof, q, b, weights)
    got = lp.cpu().numpy().T.astype(np.float64)
    ref = pr.scores(fam.counts, prof.a, prof.w, S, b, q.offsets, q.deadline, q.now, weights, store_fp32=True)
    assert got.shape == ref.shape
    ninf = ref == -np.inf
    assert (np.isneginf(got) == ninf).all(), int((np.isneginf(got) != ninf).sum())
    err = np.abs(got[~ninf] - ref[~ninf])
    assert (err <= _tol(ref[~ninf])).all(), float(err.max())
    import _parity as par
    par.record("priority_tolerance_use", label=f"{name}/b{b_scale}",
               max_err_over_tol=float((err / _tol(ref[~ninf])).max()), max_abs_err=float(err.max()))
    exact = pr.scores(fam.counts, prof.a, prof.w, S, b, q.offsets, q.deadline, q.now, weights)
    assert ((exact == -np.inf) == ninf).all()
    # against the paper's Eq. 2 on the real (exact-count) histograms: the GPU
    # error is its arithmetic (above) plus what the store format itself does
    # (oracle.priority.store_rounding_log_priority_bound, pinned on CPU)
    off = np.asarray(q.offsets) - int(q.offsets[0])
    sig = np.empty(int(off[-1]))
    for qq in range(len(off) - 1):
        sig[off[qq]:off[qq + 1]] = np.asarray(q.deadline[off[qq]:off[qq + 1]]) - int(q.now[qq])
    worst, unbounded = 0.0, 0
    for bs in range(1, S + 1):
        bnd = pr.store_rounding_log_priority_bound(fam.counts, float(prof.a[bs - 1]), float(prof.w[bs - 1]), b, sig,
                                                   bs, weights)
        fin = np.isfinite(exact[:, bs - 1])
        ok = fin & np.isfinite(bnd)
        e = np.abs(got[ok, bs - 1] - exact[ok, bs - 1])
        assert (e <= bnd[ok] + _tol(exact[ok, bs - 1])).all(), (bs, float((e - bnd[ok]).max()))
        worst = max(worst, float(e.max()) if e.size else 0.0)
        unbounded += int((fin & ~np.isfinite(bnd)).sum())
    import _parity as par
    par.record("priority_vs_exact", label=f"{name}/b{b_scale}", elements=int(np.isfinite(exact).sum()),
               max_abs_log_err=worst, unbounded_elements=unbounded)


def test_store_is_the_rounded_model():
    """The store the priority tables read holds RN32(log2 F) of the exact counts
    (the oracle's store_fp32 model) bit for bit, except within 2^-45 of a
    rounding midpoint (both sides round an fp64 log2 whose last place may
    differ)."""
    for name in ("skipnet", "rdi", "gpt"):
        fam, _, _ = _case(name, gen.SEED_BASE + 912)
        store = orj.HistogramStore.from_counts(fam.counts, fam.bin_ticks)
        got = store.log2_cdf.cpu().numpy()
        c = np.asarray(fam.counts, np.float64)
        with np.errstate(divide="ignore"):
            x = np.log2(np.cumsum(c, axis=1) / c.sum(axis=1, keepdims=True))
        ref = x.astype(np.float32)
        diff = got != ref
        if diff.any():
            lo, hi = np.minimum(got, ref).astype(np.float64), np.maximum(got, ref).astype(np.float64)
            mid = (lo + hi) / 2
            assert (np.abs(x[diff] - mid[diff]) <= 2.0 ** -45 * np.abs(x[diff])).all(), name
            assert (np.abs(got[diff].view(np.int32) - ref[diff].view(np.int32)) == 1).all()


def test_scores_queue_window_and_empty():
    fam, prof, q = _case("gpt", gen.SEED_BASE + 911, Q=24)
    b = 1.0 / fam.mean_ticks()
    store = orj.HistogramStore.from_counts(fam.counts, fam.bin_ticks)
    p = orj.LatencyProfile(prof.a, prof.w)
    tab = orj.PriorityTable(store, p, S, b)
    full = wl.device_queues(q)
    lp_full = tab.scores(full)
    # queues 5..16 through offsets that start at member offsets[5]
    o0, o1 = int(q.offsets[5]), int(q.offsets[17])
    sub = orj.Queues(full.offsets[5:18].contiguous(), full.deadline[o0:o1].contiguous(),
                     full.dist[o0:o1].contiguous(), full.now[5:17].contiguous())
    lp_sub = tab.scores(sub)
    torch.cuda.synchronize()
    assert torch.equal(lp_sub, lp_full[:, o0:o1])
    empty = orj.Queues.from_numpy(np.zeros(1, np.int64), np.zeros(0), np.zeros(0), np.zeros(0))
    assert tab.scores(empty).numel() == 0


def test_table_properties():
    fam, prof, _ = _case("rdi", gen.SEED_BASE + 912)
    b = 1.0 / fam.mean_ticks()
    store = orj.HistogramStore.from_counts(fam.counts, fam.bin_ticks)
    tab = orj.PriorityTable(store, orj.LatencyProfile(prof.a, prof.w), S, b)
    torch.cuda.synchronize()
    EL = np.exp(tab.log_expected.cpu().numpy())
    ref = np.array([pr.expected_latency(pr.batch_latency_pmf(fam.counts, bs, store_fp32=True), prof.a[bs - 1],
                                        prof.w[bs - 1])
                    for bs in range(1, S + 1)])
    assert np.allclose(EL, ref, rtol=1e-12, atol=0)
    C = tab.log_table[:, 0].cpu().numpy()
    assert (C[:, 1:] >= C[:, :-1]).all()  # prefix of non-negative terms
    assert (C[:, 0] == -np.inf).all() and np.isfinite(C[:, -1]).all()


def test_invalid_arguments():
    fam, prof, _ = _case("gpt", gen.SEED_BASE + 913)
    store = orj.HistogramStore.from_counts(fam.counts, fam.bin_ticks)
    p = orj.LatencyProfile(prof.a, prof.w)
    for bad in (dict(num_sizes=0, b_per_tick=1e-3), dict(num_sizes=S + 1, b_per_tick=1e-3),
                dict(num_sizes=4, b_per_tick=0.0), dict(num_sizes=4, b_per_tick=1e9)):
        with pytest.raises(orj.OrlojError):
            orj.PriorityTable(store, p, **bad)


def _pop_case(seed, Q=300):
    rng = np.random.default_rng(seed)
    lengths = rng.integers(0, 320, Q)
    lengths[:4] = (0, 1, 256, 319)
    off = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    N = int(off[-1])
    v = rng.integers(-40, 40, size=(N, S)).astype(np.float32) * np.float32(0.25)  # many exact ties
    v[rng.random((N, S)) < 0.2] = -np.inf
    v[rng.random((N, S)) < 0.02] = np.nan
    v[rng.random((N, S)) < 0.05] = np.float32(-0.0)
    bs = rng.integers(-1, S + 3, Q).astype(np.int32)
    bs[:8] = (1, 32, 32, 32, 0, S + 1, 5, 17)
    return off, v, bs


def test_pop_batch_bitexact():
    off, v, bs = _pop_case(gen.SEED_BASE + 914)
    Q = len(bs)
    q = orj.Queues.from_numpy(off, np.zeros(off[-1]), np.zeros(off[-1]), np.zeros(Q))
    fam = gen.gpt_family(gen.SEED_BASE + 915)
    store = orj.HistogramStore.from_counts(fam.counts, fam.bin_ticks)
    prof = gen.eq3_half(fam, S)
    tab = orj.PriorityTable(store, orj.LatencyProfile(prof.a, prof.w), S, 1e-4)
    sel = tab.pop(q, torch.from_numpy(np.ascontiguousarray(v.T)).cuda(), torch.from_numpy(bs).cuda()).cpu().numpy()
    for qi in range(Q):
        want = pr.pop_batch(v[off[qi]:off[qi + 1]], int(bs[qi]), S)
        got = [int(x) for x in sel[qi] if x >= 0]
        assert got == want, qi
        assert (sel[qi, len(got):] == -1).all()


def test_scores_then_pop_selects_the_top():
    """End to end: GPU scores -> GPU PopBatch selects members whose oracle
    priority is within the score tolerance of the oracle's top-bs (several
    selections are correct under ties, A9-style: compare the unique part)."""
    fam, prof, q = _case("skipnet", gen.SEED_BASE + 916)
    b = 1.0 / fam.mean_ticks()
    tab, qs, lp = _gpu_scores(fam, prof, q, b)
    rng = np.random.default_rng(gen.SEED_BASE + 917)
    bs = rng.integers(1, S + 1, q.Q).astype(np.int32)
    sel = tab.pop(qs, lp, torch.from_numpy(bs).cuda()).cpu().numpy()
    ref = pr.scores(fam.counts, prof.a, prof.w, S, b, q.offsets, q.deadline, q.now, store_fp32=True)
    for qi in range(q.Q):
        rows = ref[q.offsets[qi]:q.offsets[qi + 1], bs[qi] - 1][:256]
        want = pr.pop_batch(ref[q.offsets[qi]:q.offsets[qi + 1]], int(bs[qi]), S)
        got = [int(x) for x in sel[qi] if x >= 0]
        assert len(got) == len(want)
        if want:
            kth = rows[want[-1]]
            assert all(rows[r] >= kth - 2 * _tol(kth) for r in got)


@pytest.mark.parametrize("name", ["skipnet", "gpt"])
def test_piecewise_step_scores_vs_oracle(name):
    """orloj_priority_scores_steps vs the oracle's sum of
    single-step priorities; each step is the single-step arithmetic (same
    tolerance per term) combined by an fp32 log-add-exp."""
    fam, prof, q = _case(name, gen.SEED_BASE + 920, Q=64)
    b = 1.0 / fam.mean_ticks()
    p99 = fam.p99_ticks()
    offs, costs = [-p99 // 4, 0, p99 // 2], [0.25, 1.0, 1.75]
    tab, qs, _ = _gpu_scores(fam, prof, q, b)
    lp = tab.scores(qs, steps=(offs, costs))
    single = tab.scores(qs, steps=([0], [1.0]))
    base = tab.scores(qs)
    torch.cuda.synchronize()
    assert torch.equal(single, base)  # one unit step is the plain priority, bit for bit
    got = lp.cpu().numpy().T.astype(np.float64)
    ref = pr.scores_steps(fam.counts, prof.a, prof.w, S, b, q.offsets, q.deadline, q.now, offs, costs,
                          store_fp32=True)
    ninf = ref == -np.inf
    assert (np.isneginf(got) == ninf).all()
    err = np.abs(got[~ninf] - ref[~ninf])
    assert (err <= 3e-6 + 2.0 ** -21 * np.abs(ref[~ninf])).all(), float(err.max())
    for bad in (([0, 0], [1.0, 2.0]), ([0, 5], [1.0, 1.0]), ([0], [0.0]), (list(range(9)), [float(i + 1) for i in range(9)])):
        with pytest.raises(orj.OrlojError):
            tab.scores(qs, steps=bad)


def _fast_path_queues(off, v, bs):
    """Queues on PopBatch's fast path (priority_kernel.cuh): every lane's best
    other key below every selectable lane head, and either no selectable
    non-head or at least bs selectable heads (order-preserving keys, -inf /
    NaN not selectable).  Host restatement of the kernel's warp-uniform test,
    used only to show both paths ran."""
    fast = np.zeros(len(bs), bool)
    for qi in range(len(bs)):
        b = int(bs[qi])
        n = int(off[qi + 1] - off[qi])
        if not 1 <= b <= S or n <= 0:
            continue
        x = np.full(256, np.nan)  # lanes past the end: below every key
        x[:min(n, 256)] = v[off[qi]:off[qi] + min(n, 256), b - 1]
        x = np.where(np.isnan(x) & (np.arange(256) < n), -np.inf, x)
        lanes = np.where(np.isnan(x), -np.inf, x).reshape(8, 32)  # slot s, lane l: member 32 s + l
        head = lanes.max(axis=0)
        other = np.sort(lanes, axis=0)[-2]
        selh = head[head > -np.inf]
        hsel = selh.min() if selh.size else np.inf
        mx2 = other.max()
        fast[qi] = mx2 < hsel and (mx2 == -np.inf or selh.size >= b)
    return fast


def test_pop_batch_fast_and_general_paths_bitexact():
    """PopBatch on queues whose priorities are unimodal over the member index
    (the top 32 a contiguous run: one head per lane, the fast path), with
    exact ties planted at the lane heads (equal keys ordered by member index),
    with a tie between a head and a second member (general path), and queues
    shorter than 32 (general path).  Bit-exact against the oracle."""
    rng = np.random.default_rng(gen.SEED_BASE + 930)
    Q = 400
    lengths = rng.integers(32, 257, Q)
    lengths[:8] = (32, 256, 256, 31, 5, 256, 256, 256)
    off = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    N = int(off[-1])
    v = np.empty((N, S), np.float32)
    for qi in range(Q):
        n = int(lengths[qi])
        r = np.arange(n)
        for s in range(S):
            peak = rng.uniform(0, n)
            v[off[qi]:off[qi + 1], s] = (-np.abs(r - peak) * rng.uniform(0.01, 0.5)).astype(np.float32)
    v[off[1]:off[2], :] = np.float32(-1.0)                   # 256 equal keys: each head ties its lane's next
    v[off[2]:off[2] + 32, :] = np.float32(-0.5)              # 32 equal heads, everything else lower
    v[off[2] + 32:off[3], :] = np.float32(-0.75)
    v[off[6]:off[8], :] = -np.inf                             # only a few selectable members:
    v[off[6] + 100:off[6] + 111, :] = np.float32(-2.0)        # 11 in distinct lanes (fast), and
    v[off[7] + 100:off[7] + 111, :] = np.float32(-2.0)
    v[off[7] + 132, :] = np.float32(-3.0)                     # one more behind a head (general)
    bs = rng.integers(1, S + 1, Q).astype(np.int32)
    bs[:8] = (32, 32, 32, 32, 3, 17, 32, 32)
    q = orj.Queues.from_numpy(off, np.zeros(N), np.zeros(N), np.zeros(Q))
    fam = gen.gpt_family(gen.SEED_BASE + 915)
    store = orj.HistogramStore.from_counts(fam.counts, fam.bin_ticks)
    prof = gen.eq3_half(fam, S)
    tab = orj.PriorityTable(store, orj.LatencyProfile(prof.a, prof.w), S, 1e-4)
    sel = tab.pop(q, torch.from_numpy(np.ascontiguousarray(v.T)).cuda(), torch.from_numpy(bs).cuda()).cpu().numpy()
    for qi in range(Q):
        want = pr.pop_batch(v[off[qi]:off[qi + 1]], int(bs[qi]), S)
        got = [int(x) for x in sel[qi] if x >= 0]
        assert got == want, qi
        assert (sel[qi, len(got):] == -1).all()
    fast = _fast_path_queues(off, v, bs)
    assert fast[2] and fast[3] and fast[6] and not fast[1] and not fast[7]
    assert 0.3 < fast.mean() < 1.0, fast.mean()
    import _parity as par
    par.record("pop_batch_paths", label="unimodal+ties", queues=Q, fast_path=int(fast.sum()))


def test_scores_vector_map_equals_scalar_map():
    """P1-shaped queues (256 members, 4-aligned starts) take the 16-byte vector
    member map; the same queues shifted by one member (a 1-member queue in
    front) take the strided map.  Same element arithmetic: bit-identical
    scores.  A sample is checked against the oracle as well."""
    cfg = gen.config_priority(Q=24, n=256)
    q = cfg.queues
    b = 1.0 / cfg.fam.mean_ticks()
    store = orj.HistogramStore.from_counts(cfg.fam.counts, cfg.fam.bin_ticks)
    p = orj.LatencyProfile(cfg.profile.a, cfg.profile.w)
    tab = orj.PriorityTable(store, p, S, b)
    lp_vec = tab.scores(wl.device_queues(q))
    off2 = np.concatenate([[0], np.asarray(q.offsets) + 1]).astype(np.int64)
    dl2 = np.concatenate([[int(q.now[0]) + 1000], np.asarray(q.deadline)]).astype(np.int64)
    dist2 = np.concatenate([[0], np.asarray(q.dist)]).astype(np.int32)
    now2 = np.concatenate([[int(q.now[0])], np.asarray(q.now)]).astype(np.int64)
    lp_sc = tab.scores(orj.Queues.from_numpy(off2, dl2, dist2, now2))
    torch.cuda.synchronize()
    assert torch.equal(lp_vec, lp_sc[:, 1:])
    got = lp_vec.cpu().numpy().T.astype(np.float64)
    sub = np.arange(0, 3)
    o = np.asarray(q.offsets)
    ref = pr.scores(cfg.fam.counts, cfg.profile.a, cfg.profile.w, S, b, o[:4], q.deadline[:o[3]], q.now[:3],
                    store_fp32=True)
    g = got[:o[3]]
    ninf = ref == -np.inf
    assert (np.isneginf(g) == ninf).all()
    assert (np.abs(g[~ninf] - ref[~ninf]) <= _tol(ref[~ninf])).all()


@pytest.mark.parametrize("b_scale", [1.0, 20.0])
def test_scores_slack_beyond_the_cap(b_scale):
    """Members whose slack exceeds the lookup's 2^30-tick cap (the warp-uniform
    slow path adds b (sigma - cap) in fp32) and members far past their deadline,
    in both tiers (b_scale 1: the fitted-polynomial tier, 20: the general one),
    in aligned full queues (vector map) and ragged ones."""
    fam = gen.gpt_family(gen.SEED_BASE + 960)
    prof = gen.eq3_half(fam, S)
    rng = np.random.default_rng(gen.SEED_BASE + 961)
    lengths = np.array([256, 256, 37, 256, 5, 256], np.int64)
    q = gen.snapshot_queues(gen.SEED_BASE + 962, lengths, fam.p99_ticks(), D=fam.D)
    o = np.asarray(q.offsets)
    dl = np.asarray(q.deadline).copy()
    for qq in range(len(lengths)):
        seg = slice(o[qq], o[qq + 1])
        far = rng.random(o[qq + 1] - o[qq]) < 0.3
        dl[seg][far] = int(q.now[qq]) + (1 << 30) + rng.integers(0, 1 << 33, far.sum())
        past = rng.random(o[qq + 1] - o[qq]) < 0.1
        dl[seg][past] = int(q.now[qq]) - rng.integers(1, 1 << 20, past.sum())
    for qq in range(len(lengths)):  # keep each queue deadline-ordered
        dl[o[qq]:o[qq + 1]] = np.sort(dl[o[qq]:o[qq + 1]])
    q.deadline = dl
    b = b_scale / fam.mean_ticks()
    _, _, lp = _gpu_scores(fam, prof, q, b)
    got = lp.cpu().numpy().T.astype(np.float64)
    ref = pr.scores(fam.counts, prof.a, prof.w, S, b, q.offsets, q.deadline, q.now, store_fp32=True)
    ninf = ref == -np.inf
    assert (np.isneginf(got) == ninf).all()
    err = np.abs(got[~ninf] - ref[~ninf])
    assert (err <= _tol(ref[~ninf])).all(), float(err.max())
