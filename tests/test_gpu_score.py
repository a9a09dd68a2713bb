"""GPU parity: orloj_score_batches / orloj_pick_batch vs the fp64 oracle.

Every test calls the CUDA library through the C ABI (paper_2209_00159_b200)
and compares element by element with oracle/ on the same seeded inputs.
Tolerances (north star): |P| <= 1e-5, |E_k| <= 1e-5 k, k*
bit-exact except documented ties; integer-valued cases bit-exact.
"""
import json
import os
from fractions import Fraction

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


def _run_all(store_counts, bin_ticks, prof, q, want_EL=True):
    store = orj.HistogramStore.from_counts(store_counts, bin_ticks)
    store.validate()
    qs = wl.device_queues(q)
    qs.validate(store)
    p = orj.LatencyProfile(prof.a, prof.w)
    sc = orj.score_batches(store, p, qs, want_P=True, want_EL=want_EL)
    # E alone takes the pick's kernel (lanes over candidate sizes for short
    # queues over a small store), so best_E must equal its E[k*] bit for bit
    e_only = orj.score_batches(store, p, qs)["E"]
    bk, bE = orj.pick_batch(store, p, qs)
    torch.cuda.synchronize()
    out = {k: (v.cpu().numpy() if v is not None else None) for k, v in sc.items()}
    out["E_only"] = e_only.cpu().numpy()
    return out, bk.cpu().numpy(), bE.cpu().numpy()


def _check_all(counts, prof, q, gpu, want_EL=True):
    sc, bk, bE = gpu
    ref = par.oracle_score(counts, prof.a, prof.w, q, want_P=True, want_EL=want_EL)
    lens = np.diff(q.offsets)
    kmax = len(prof.a)
    par.check_E(sc["E"], ref["E"], lens, kmax)
    e_pick = sc.get("E_only", sc["E"])   # the E of the pick's kernel
    par.check_E(e_pick, ref["E"], lens, kmax)
    par.check_P(sc["P"], ref["P"], lens, kmax)
    ties = par.check_pick(bk, bE, e_pick, ref["E"], ref["best_k"], lens, kmax)
    if want_EL:
        K = np.minimum(lens, kmax)
        B = counts.shape[1]
        w = np.asarray(prof.w, np.float64)
        valid = np.arange(1, kmax + 1)[None, :] <= K[:, None]
        # E[L_B] = a + w E[max bin]; E[max bin] carries <= 1e-5 per bin
        tol = w[None, :] * (1e-5 * B) + 1e-6 * np.abs(ref["EL"]) + 1.0
        err = np.abs(sc["EL"].astype(np.float64) - ref["EL"])
        assert (err[valid] <= np.broadcast_to(tol, err.shape)[valid]).all(), err[valid].max()
        assert (sc["EL"][~valid] == 0).all()
    return ties


def test_config1_vs_oracle_and_bruteforce():
    c = gen.config1()
    gpu = _run_all(c.fam.counts, c.fam.bin_ticks, c.profile, c.queues)
    _check_all(c.fam.counts, c.profile, c.queues, gpu)
    q = c.queues
    Pb, Eb = oracle.bruteforce(c.fam.counts, c.profile.a, c.profile.w, q.deadline, q.dist, int(q.now[0]))
    assert np.abs(gpu[0]["E"][0] - Eb).max() <= 1e-5 * 8
    assert np.abs(gpu[0]["P"][0] - Pb).max() <= 1e-5
    assert gpu[1][0] == int(np.argmax(Eb)) + 1


def _appendix():
    with open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("ex", _appendix()["examples"], ids=lambda e: e["name"])
def test_appendix_a(ex):
    g = _appendix()
    counts = np.array(ex["counts"], np.uint32)
    K = len(ex["deadline"])
    q = gen.Queues(np.array([0, K], np.int64), np.zeros(K, np.int64), np.array(ex["deadline"], np.int64),
                   np.arange(K, dtype=np.int32), np.array([g["now"]], np.int64))
    prof = gen.Profile(np.array(g["a"], np.int64), np.array(g["w"], np.int64))
    sc, bk, bE = _run_all(counts, 1, prof, q)
    E = np.array([float(Fraction(x)) for x in ex["E"]])
    assert np.abs(sc["E"][0] - E).max() <= 1e-6
    assert np.abs(sc["E_only"][0] - E).max() <= 1e-6
    assert bk[0] == ex["k_star"]          # includes Ex3's exact tie -> smallest k


def test_config2_full():
    c = gen.config2()
    ties = _check_all(c.fam.counts, c.profile, c.queues, _run_all(c.fam.counts, c.fam.bin_ticks, c.profile, c.queues))
    par.record("pick_ties", label="C2-full", queues=c.queues.Q, differing_choices=ties)
    assert ties <= 2


@pytest.mark.parametrize("near", [False, True])
def test_config4_full(near):
    """1,048,576 decisions.  Exact point masses: E_k are integers and k* must
    equal the constant-latency planner (and the oracle) bit for bit."""
    c = gen.config4(near=near)
    q = c.queues
    store = orj.HistogramStore.from_counts(c.fam.counts, c.fam.bin_ticks)
    p = orj.LatencyProfile(c.profile.a, c.profile.w)
    qs = wl.device_queues(q)
    bk, bE = orj.pick_batch(store, p, qs)
    torch.cuda.synchronize()
    bk, bE = bk.cpu().numpy(), bE.cpu().numpy()
    ref = par.oracle_score(c.fam.counts, c.profile.a, c.profile.w, q)
    if not near:
        assert (bk == ref["best_k"]).all()
        assert (bE.astype(np.float64) == ref["best_E"]).all()
        # textbook planner, integers only: E_k = #{r <= k: now + a_k + w_k M_k <= D_r}
        n, S = 32, 1 << 16          # planner on the first 65,536 queues (host memory)
        m_of = np.array([int(np.argmax(r)) + 1 for r in c.fam.counts])
        M = np.maximum.accumulate(m_of[q.dist[:S * n].reshape(-1, n)], axis=1)
        dur = c.profile.a[None, :] + c.profile.w[None, :] * M
        ok = (q.now[:S, None, None] + dur[:, :, None]) <= q.deadline[:S * n].reshape(-1, n)[:, None, :]
        ok &= np.tri(n, dtype=bool)[None, :, :]
        Ek = ok.sum(2)
        assert (bk[:S] == Ek.argmax(1) + 1).all()
    else:
        sc = orj.score_batches(store, p, qs)
        torch.cuda.synchronize()
        E = sc["E"].cpu().numpy()
        lens = np.diff(q.offsets)
        par.check_E(E, ref["E"], lens, 32)
        ties = par.check_pick(bk, bE, E, ref["E"], ref["best_k"], lens, 32)
        agree = (bk == ref["best_k"]).mean()
        par.record("pick_ties", label="C4-near-full", queues=len(bk), differing_choices=ties)
        assert agree > 0.9999, agree
        assert ties < 1e-4 * len(bk)


@pytest.mark.parametrize("kmax", [256, 64])
def test_config3_shape_small(kmax):
    """C3 rows (per-request, permuted 1 KB gathers) at 512 queues x 256 members:
    full E / P / E[L_B] parity at the bench's kernel variant (B = 256, 32-byte
    row loads, kmax up to 256)."""
    cfg = gen.config3(Q=512, n=256, kmax=kmax, T=256)
    store = wl.c3_store(cfg)
    q = cfg.queues
    p = orj.LatencyProfile(cfg.profile.a, cfg.profile.w)
    qs = wl.device_queues(q)
    sc = orj.score_batches(store, p, qs, want_P=True, want_EL=True)
    bk, bE = orj.pick_batch(store, p, qs)
    torch.cuda.synchronize()
    rows = gen.rows_host(cfg.row_seed, np.arange(cfg.n_rows, dtype=np.uint64), cfg.fam.counts)
    gpu = ({k: v.cpu().numpy() for k, v in sc.items()}, bk.cpu().numpy(), bE.cpu().numpy())
    _check_all(rows, cfg.profile, q, gpu)


def test_config3_full_size_stream():
    """The bench's launch: C3 at full size (65,536 queues x 256, 16.8 M rows,
    17.2 GB store, so the TMA ring runs its STREAM variant: L1 bypass,
    L2 evict-first).  k* of all queues comes from the bench's pick call; a
    4,096-queue chunk in the middle (SURVEY §8(d) subset) is scored by the
    STREAM score kernel over the same full store (queue offsets with a base,
    include/orloj.h) and checked element by element against the oracle: E, P,
    E[L_B] and the pick's k* (documented ties counted and bounded)."""
    cfg = gen.config3()
    store = wl.c3_store(cfg)
    assert store.log2_cdf.numel() * 4 > 256 << 20            # > STREAM_STORE_BYTES: the streaming variant
    q = cfg.queues
    p = orj.LatencyProfile(cfg.profile.a, cfg.profile.w)
    qs = wl.device_queues(q, with_arrival=False)
    bk, bE = orj.pick_batch(store, p, qs)
    torch.cuda.synchronize()
    bk, bE = bk.cpu().numpy(), bE.cpu().numpy()
    q0, nq = 30_000, 4096
    m0, m1 = int(q.offsets[q0]), int(q.offsets[q0 + nq])
    chunk = orj.Queues(qs.offsets[q0:q0 + nq + 1], qs.deadline[m0:m1], qs.dist[m0:m1], qs.now[q0:q0 + nq])
    sc = orj.score_batches(store, p, chunk, want_P=True, want_EL=True)
    torch.cuda.synchronize()
    gpu_sc = {k: v.cpu().numpy() for k, v in sc.items()}
    del sc, store, qs
    torch.cuda.empty_cache()
    sub = q.subset(np.arange(q0, q0 + nq))
    rows = gen.rows_host(cfg.row_seed, sub.dist.astype(np.uint64), cfg.fam.counts)
    local = gen.Queues(sub.offsets, sub.arrival, sub.deadline, np.arange(len(sub.dist), dtype=np.int32), sub.now)
    ties = _check_all(rows, cfg.profile, local, (gpu_sc, bk[q0:q0 + nq], bE[q0:q0 + nq]))
    par.record("pick_ties", label="C3-full-stream-4096", queues=nq, differing_choices=ties)
    assert ties <= 1e-3 * nq, ties


def _random_queues(seed, Q, D, B, kmax, maxlen):
    rng = np.random.default_rng(seed)
    counts = np.stack([gen.largest_remainder(rng.dirichlet(np.ones(B) * rng.uniform(0.2, 2))) for _ in range(D)])
    counts[rng.random((D, B)) < 0.3] = 0
    counts[:, rng.integers(0, B, D)] += 7
    a = np.cumsum(rng.integers(0, 50, kmax)).astype(np.int64)
    w = np.cumsum(rng.integers(0, 4, kmax)).astype(np.int64) + rng.integers(1, 30)
    lens = rng.integers(0, maxlen + 1, Q)
    lens[:3] = [0, 1, maxlen]
    horizon = int(a[-1] + w[-1] * B)
    now = (rng.integers(0, 1 << 62, Q) // 2).astype(np.int64)
    dl = []
    for qq in range(Q):
        s = rng.integers(-horizon // 8, horizon + horizon // 4, lens[qq])
        # put a third of the members exactly on bin boundaries of some k
        kk = rng.integers(0, kmax, lens[qq])
        mm = rng.integers(0, B + 1, lens[qq])
        edge = a[kk] + w[kk] * mm + rng.integers(-1, 2, lens[qq])
        s = np.where(rng.random(lens[qq]) < 0.33, edge, s)
        dl.append(np.sort(now[qq] + s))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    dl = np.concatenate(dl).astype(np.int64) if Q else np.zeros(0, np.int64)
    q = gen.Queues(off, dl - 10, dl, rng.integers(0, D, off[-1]).astype(np.int32), now)
    return counts.astype(np.uint32), gen.Profile(a, w), q


@pytest.mark.parametrize("B,kmax,maxlen", [(4, 1, 3), (12, 5, 9), (32, 32, 40), (36, 33, 70), (64, 100, 130),
                                           (100, 64, 64), (132, 200, 260), (256, 256, 300), (252, 96, 120),
                                           (20, 32, 45), (40, 32, 50), (52, 17, 30), (64, 32, 31)])
def test_ragged_edges(B, kmax, maxlen):
    """Empty and ragged queues, n < kmax and n > kmax, B % 8 == 4 (half row
    vectors), every bins-per-lane / slot variant, sigma on exact bin edges and
    +-1 tick, negative and huge slack, absolute times near 2^61.  The last four
    shapes (kmax <= 32, B <= 64) run the short-queue pick with one and two bins
    per lane and B below a whole number of lanes."""
    counts, prof, q = _random_queues(B * 1000 + kmax, Q=67, D=9, B=B, kmax=kmax, maxlen=maxlen)
    _check_all(counts, prof, q, _run_all(counts, 1, prof, q))


def test_point_mass_lookup_exact():
    """Bin lookups are exact integers: with point masses P is exactly 0 or 1 and
    flips exactly at sigma = a_k + w_k m (inclusive deadline, A11)."""
    B, kmax = 64, 40
    counts = np.zeros((B, B), np.uint32)
    counts[np.arange(B), np.arange(B)] = 5
    rng = np.random.default_rng(11)
    a = np.cumsum(rng.integers(0, 1000, kmax)).astype(np.int64)
    w = np.cumsum(rng.integers(0, 300, kmax)).astype(np.int64) + 977
    Q = 300
    lens = rng.integers(1, kmax + 1, Q)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    now = rng.integers(0, 1 << 50, Q).astype(np.int64)
    dl, dist = [], []
    for qq in range(Q):
        k = lens[qq]
        m = rng.integers(1, B + 1, k)
        s = np.sort(a[k - 1] + w[k - 1] * rng.integers(0, B + 1, k) + rng.integers(-1, 2, k))
        dl.append(now[qq] + s)
        dist.append(m - 1)
    q = gen.Queues(off, np.concatenate(dl) - 1, np.concatenate(dl).astype(np.int64),
                   np.concatenate(dist).astype(np.int32), now)
    prof = gen.Profile(a, w)
    sc, bk, bE = _run_all(counts, 1, prof, q, want_EL=False)
    ref = par.oracle_score(counts, a, w, q, want_P=True)
    K = np.minimum(lens, kmax)
    tri = np.concatenate([np.full(k, k) for k in range(1, kmax + 1)])
    valid = tri[None, :] <= K[:, None]
    assert (sc["P"][valid] == ref["P"][valid]).all()
    assert (sc["E"] == ref["E"]).all()
    assert (sc["E_only"] == ref["E"]).all()
    assert (bk == ref["best_k"]).all()


def test_errors():
    B = 8
    counts = np.ones((2, B), np.uint32)
    bad = counts.copy()
    bad[1] = 0
    with pytest.raises(orj.OrlojError) as ei:
        orj.HistogramStore.from_counts(bad, 1)
    assert ei.value.status == 2                                      # COLD_START
    store = orj.HistogramStore.from_counts(counts, 1)
    q = wl.device_queues(gen.Queues(np.array([0, 2], np.int64), np.zeros(2, np.int64), np.array([5, 3], np.int64),
                                    np.zeros(2, np.int32), np.zeros(1, np.int64)))
    with pytest.raises(orj.OrlojError) as ei:
        q.validate(store)
    assert ei.value.status == 3                                      # UNSORTED
    with pytest.raises(orj.OrlojError) as ei:
        orj.pick_batch(store, orj.LatencyProfile([2, 1], [1, 1]), q)
    assert ei.value.status == 1                                      # non-monotone profile
    with pytest.raises(orj.OrlojError) as ei:
        orj.pick_batch(store, orj.LatencyProfile([0], [1 << 29]), q)
    assert ei.value.status == 4                                      # horizon > 2^31 ticks
    with pytest.raises(orj.OrlojError) as ei:
        orj.pick_batch(store, orj.LatencyProfile(np.zeros(257), np.ones(257)), q)
    assert ei.value.status == 4                                      # kmax > 256
    qd = wl.device_queues(gen.Queues(np.array([0, 1], np.int64), np.zeros(1, np.int64), np.zeros(1, np.int64),
                                     np.array([5], np.int32), np.zeros(1, np.int64)))
    with pytest.raises(orj.OrlojError) as ei:
        qd.validate(store)
    assert ei.value.status == 1                                      # dist id out of range


def test_empty_and_host_path():
    """Q = 0 is a no-op; the end-to-end host entry point equals the device one."""
    c = gen.config2(Q=300)
    store = orj.HistogramStore.from_counts(c.fam.counts, c.fam.bin_ticks)
    p = orj.LatencyProfile(c.profile.a, c.profile.w)
    e = wl.device_queues(gen.Queues(np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64),
                                    np.zeros(0, np.int32), np.zeros(0, np.int64)))
    bk0, _ = orj.pick_batch(store, p, e)
    assert bk0.numel() == 0
    q = c.queues
    bk, bE = orj.pick_batch(store, p, wl.device_queues(q))
    pin = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).pin_memory()  # noqa: E731
    hargs = (pin(q.offsets, np.int64), pin(q.deadline, np.int64), pin(q.dist, np.int32), pin(q.now, np.int64))
    pageable = tuple(torch.from_numpy(np.ascontiguousarray(a.numpy())) for a in hargs)
    # (1, 1): 230 KB per call -> copies; (5, 2) and (300, 3): <= 64 KiB per call
    # -> zero-copy (mapped pinned memory), or copies for pageable host arrays
    for chunks, streams, args in ((1, 1, hargs), (5, 2, hargs), (300, 3, hargs), (300, 3, pageable)):
        hp = orj.HostPicker(store, p, q.offsets, chunks=chunks, streams=streams)
        hk, hE = hp.pick(*args)
        torch.cuda.synchronize()
        assert (hk.numpy() == bk.cpu().numpy()).all() and (hE.numpy() == bE.cpu().numpy()).all()
    # queue offsets may start at any base (a chunk of a larger queue set)
    sub = orj.Queues(wl.t(q.offsets[100:201], np.int64), wl.t(q.deadline[q.offsets[100]:q.offsets[200]], np.int64),
                     wl.t(q.dist[q.offsets[100]:q.offsets[200]], np.int32), wl.t(q.now[100:200], np.int64))
    sk, sE = orj.pick_batch(store, p, sub)
    torch.cuda.synchronize()
    assert (sk.cpu().numpy() == bk.cpu().numpy()[100:200]).all()


def test_store_build_values():
    """log2_cdf rows: 0.0f exactly at the last bin, -inf exactly where F = 0, and
    2^row within fp32 rounding of the oracle's fp64 CDF."""
    fam = gen.skipnet_family(9)
    counts = fam.counts.copy()
    counts[0, :5] = 0
    counts[0, 5] += 1
    st = orj.HistogramStore.from_counts(counts, fam.bin_ticks)
    torch.cuda.synchronize()
    L = st.log2_cdf.cpu().numpy().astype(np.float64)
    F = oracle.cdf(counts)
    assert (L[:, -1] == 0.0).all()
    assert ((L == -np.inf) == (F == 0)).all()
    nz = F > 0
    assert np.abs(np.exp2(L[nz]) - F[nz]).max() <= 1e-6


@pytest.mark.parametrize("B,kmax,maxlen", [(16, 8, 12), (64, 40, 70), (100, 64, 64), (132, 130, 140),
                                           (40, 20, 30), (64, 32, 45)])
def test_tma_row_path(B, kmax, maxlen):
    """Per-request rows (store > 48 KiB, so rows come through the TMA ring
    rather than the shared-memory store) for every bins-per-lane variant; with
    kmax <= 32 and B <= 64 the pick and E-only score take the short-queue
    kernel reading its rows from global memory (one and two bins per lane)."""
    counts, prof, q = _random_queues(7 * B + kmax, Q=97, D=9, B=B, kmax=kmax, maxlen=maxlen)
    rng = np.random.default_rng(B)
    D = max(9, (64 << 10) // (4 * B) + 1)
    big = counts[rng.integers(0, counts.shape[0], D)]
    q.dist[:] = rng.integers(0, D, len(q.dist)).astype(np.int32)
    assert big.size * 4 > (48 << 10)
    _check_all(big, prof, q, _run_all(big, 1, prof, q))
