"""GPU parity of K1 (lens), normalisation, K2 (cover binning) and the exact
fp64 distance orders — bit-exact against the oracle / numpy / scipy."""

import numpy as np
import pytest
from scipy.spatial.distance import cdist

from oracle import mapper_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_2011_03209_b200.device import require_gpu

    return require_gpu()


def _dev(x, dev):
    from paper_2011_03209_b200.device import to_device_f64

    return to_device_f64(x, dev)


@pytest.mark.parametrize("d", [1, 2, 3, 7, 8, 9, 15, 16, 31, 64, 100, 128, 129, 136, 200, 250, 256,
                               257, 264, 384, 500, 512, 1000, 2048])
def test_lens_bit_exact(dev, d):
    from paper_2011_03209_b200 import engine, _native

    rng = np.random.default_rng(d)
    X = rng.standard_normal((777, d)) * rng.uniform(0.01, 1e3)
    X[5] = 0.0
    X[6, 0] = -0.0
    Xd = _dev(X, dev)
    assert np.array_equal(engine.lens(Xd, _native.LENS_L2).cpu().numpy(),
                          np.sqrt((X ** 2).sum(axis=1)))
    assert np.array_equal(engine.lens(Xd, _native.LENS_LINF).cpu().numpy(),
                          np.abs(X).max(axis=1))
    assert np.array_equal(engine.lens(Xd, _native.LENS_COLUMN, d - 1).cpu().numpy(), X[:, d - 1])


@pytest.mark.parametrize("n", [1, 2, 3, 5])
@pytest.mark.parametrize("d", [64, 256, 512])
def test_lens_few_rows(dev, n, d):
    """Rows packed 4 / 2 / 1 per warp: the tail of a row count not divisible
    by the packing must be written exactly once."""
    from paper_2011_03209_b200 import engine, _native

    X = np.random.default_rng(n * d).standard_normal((n, d))
    assert np.array_equal(engine.lens(_dev(X, dev), _native.LENS_L2).cpu().numpy(),
                          np.sqrt((X ** 2).sum(axis=1)))


def test_lens_large_rows(dev):
    from paper_2011_03209_b200 import engine, _native

    rng = np.random.default_rng(1)
    X = rng.standard_normal((200_000, 256))
    got = engine.lens(_dev(X, dev), _native.LENS_L2).cpu().numpy()
    assert np.array_equal(got, np.sqrt((X ** 2).sum(axis=1)))


@pytest.mark.parametrize("scheme", ["minmax", "l2"])
@pytest.mark.parametrize("d", [1, 5, 64, 300])
def test_normalize_bit_exact(dev, scheme, d):
    from paper_2011_03209_b200 import engine

    rng = np.random.default_rng(d)
    X = rng.standard_normal((501, d)) * 5 + 3
    X[3] = 0.0
    if d > 1:
        X[:, 1] = 2.5  # constant column -> span 1
    got = engine.normalize(_dev(X, dev), scheme).cpu().numpy()
    assert np.array_equal(got, O.normalize(X, scheme))


def _gpu_membership(values, n, p, dev):
    from paper_2011_03209_b200 import FilterSpec, FilterValues, build_cover, engine

    arr = np.asarray(values, dtype=np.float64)
    if arr.ndim == 1:
        arr = arr[:, None]
    fv = FilterValues(values=arr.copy(), specs=[FilterSpec(kind="l2-norm")] * arr.shape[1])
    cover = build_cover(fv, n, p)
    rows, offs = engine.membership(_dev(arr, dev), cover)
    r = rows.cpu().numpy()
    got = [r[offs[k]:offs[k + 1]].tolist() for k in range(len(offs) - 1)]
    axes = [[(iv.lo, iv.hi) for iv in ax] for ax in cover.axes]
    want = [m.tolist() for m in O.membership(arr, axes)]
    return got, want


@pytest.mark.parametrize("seed", range(25))
def test_membership_matches_oracle_1d(dev, seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 30_000))
    v = rng.standard_normal(N) * rng.uniform(0.01, 100)
    if seed % 3 == 0:
        v = np.round(v, 1)  # many duplicates / values on endpoints
    n = int(rng.integers(1, 60))
    p = float(rng.uniform(0, 0.95))
    got, want = _gpu_membership(v, [n], [p], dev)
    assert got == want


@pytest.mark.parametrize("seed", range(10))
def test_membership_matches_oracle_2d(dev, seed):
    rng = np.random.default_rng(100 + seed)
    N = int(rng.integers(1, 20_000))
    v = rng.standard_normal((N, 2)) * rng.uniform(0.1, 10, 2)
    n = [int(x) for x in rng.integers(1, 16, 2)]
    p = [float(x) for x in rng.uniform(0, 0.9, 2)]
    got, want = _gpu_membership(v, n, p, dev)
    assert got == want


@pytest.mark.parametrize("n", [[300], [20, 25], [16, 16], [17, 16]])
def test_membership_many_elements(dev, n):
    """Element counts around and above the shared-memory cursor limit (256)."""
    rng = np.random.default_rng(sum(n))
    m = len(n)
    v = rng.standard_normal((40_000, m)) if m == 2 else rng.standard_normal(40_000)
    got, want = _gpu_membership(v, n, [0.4] * m, dev)
    assert got == want


def test_membership_boundary_and_degenerate(dev):
    got, want = _gpu_membership([0.0, 0.5, 1.0], [2], [0.0], dev)  # test_cover.py:56-61
    assert got == [[0, 1], [1, 2]] == want
    with pytest.warns(UserWarning):
        got, want = _gpu_membership([4.0, 4.0, 4.0], [5], [0.3], dev)
    assert got == [[0, 1, 2]] == want
    v = np.linspace(0.0, 1.0, 101)  # test_cover.py:64-74
    got, want = _gpu_membership(v, [6], [0.3], dev)
    assert got == want


def test_membership_nan_is_in_nothing(dev):
    v = np.array([0.0, np.nan, 1.0, 0.5])
    from paper_2011_03209_b200 import FilterSpec, FilterValues, engine
    from paper_2011_03209_b200.cover import Cover, Interval

    cover = Cover(n=[2], p=[0.0], axes=[[Interval(0.0, 0.5, 0, 0), Interval(0.5, 1.0, 0, 1)]],
                  filter_range=[(0.0, 1.0)])
    rows, offs = engine.membership(_dev(v[:, None], dev), cover)
    r = rows.cpu().numpy()
    assert r[offs[0]:offs[1]].tolist() == [0, 3] and r[offs[1]:offs[2]].tolist() == [2, 3]


@pytest.mark.parametrize("d", [1, 2, 3, 16, 64, 127, 128, 129, 256, 300])
def test_exact_distance_orders(dev, d):
    from paper_2011_03209_b200 import from_array, pairwise_distances, _native

    rng = np.random.default_rng(d)
    X = rng.standard_normal((150, d)) * 4
    pc = from_array(X)
    rows = np.arange(0, 150, 2)
    seq = pairwise_distances(pc, rows, order=_native.ORDER_SEQUENTIAL)
    assert np.array_equal(seq, cdist(X[rows], X[rows]))
    pw = pairwise_distances(pc, rows, order=_native.ORDER_PAIRWISE)
    P = X[rows]
    ref = np.stack([np.sqrt(((P - P[i]) * (P - P[i])).sum(axis=1)) for i in range(len(rows))])
    assert np.array_equal(pw, ref)


@pytest.mark.parametrize("sizes", [[1, 7, 8, 129, 1000], [250_001, 3, 131_072]])
def test_node_payload_matches_numpy(dev, sizes):
    """bm_node_stats: per-column means (numpy axis-0 mean: sequential row sum)
    and filter means (1-D mean: pairwise sum) bit-exact, including nodes of
    several hundred thousand rows (deep pairwise recursion)."""
    import torch

    from paper_2011_03209_b200 import engine as eng

    rng = np.random.default_rng(sum(sizes))
    n, d, m = 600_000, 5, 2
    X = rng.standard_normal((n, d)) * 1e3
    F = rng.standard_normal((n, m)) * 1e6
    rows = [np.sort(rng.choice(n, s, replace=False)) for s in sizes]
    off = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    flat = np.concatenate(rows)
    st, fm = eng.node_payload(torch.from_numpy(X).to(dev), torch.from_numpy(F).to(dev),
                              torch.from_numpy(flat).to(dev), torch.from_numpy(off).to(dev),
                              len(sizes))
    st, fm = st.cpu().numpy(), fm.cpu().numpy()
    for v, r in enumerate(rows):
        assert np.array_equal(st[v], X[r].mean(axis=0)), v
        for a in range(m):
            assert fm[v, a] == F[r, a].mean(), (v, a)
