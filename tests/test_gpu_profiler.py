"""GPU: online profiler (orloj_histogram_accumulate) vs the plain definition —
bin i = clamp(ceil(solo / Delta), 1, B) per sample, counted with numpy — and a
window reset + store refresh that reproduces a store built from the same
counts directly."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2209_00159_b200 as orj  # noqa: E402


def _expected(dist, solo, D, B, delta):
    out = np.zeros((D, B), np.int64)
    for d, x in zip(dist, solo):
        if 0 <= d < D:
            i = max(1, min(B, -(-int(x) // delta) if x > 0 else 1))
            out[d, i - 1] += 1
    return out


@pytest.mark.parametrize("D,B,n", [(8, 64, 50_000), (3, 16, 7), (500, 256, 200_000)])
def test_accumulate_matches_definition(D, B, n):
    rng = np.random.default_rng(D * B + n)
    delta = int(rng.integers(50, 5000))
    dist = rng.integers(-1, D + 1, n).astype(np.int32)               # includes out-of-range ids (ignored)
    solo = rng.integers(0, delta * (B + 5), n).astype(np.int64)
    solo[: min(n, 5)] = [0, 1, delta, delta + 1, delta * B][: min(n, 5)]  # exact bin edges
    prof = orj.Profiler(D, B, delta)
    half = n // 2
    prof.add(torch.from_numpy(dist[:half]).cuda(), torch.from_numpy(solo[:half]).cuda())
    prof.add(torch.from_numpy(dist[half:]).cuda(), torch.from_numpy(solo[half:]).cuda())
    torch.cuda.synchronize()
    assert (prof.counts.cpu().numpy().astype(np.int64) == _expected(dist, solo, D, B, delta)).all()


def test_window_reset_and_refresh():
    D, B, delta = 4, 32, 100
    rng = np.random.default_rng(1)
    dist = rng.integers(0, D, 10_000).astype(np.int32)
    solo = rng.integers(1, delta * B, 10_000).astype(np.int64)
    prof = orj.Profiler(D, B, delta)
    prof.add(torch.from_numpy(dist).cuda(), torch.from_numpy(solo).cuda())
    store = orj.HistogramStore.empty(D, B, delta)
    prof.refresh(store)
    exp = _expected(dist, solo, D, B, delta)
    L = store.log2_cdf.cpu().numpy().astype(np.float64)
    F = oracle.cdf(exp.astype(np.uint32))
    assert np.abs(np.exp2(L) - F).max() <= 1e-6 and (L[:, -1] == 0).all()
    prof.reset()
    torch.cuda.synchronize()
    assert int(prof.counts.sum()) == 0
