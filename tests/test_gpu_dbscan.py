"""GPU parity of K3..K6 (per-element DBSCAN) — mirrors the reference's
test_clustering.py cases and checks randomized instances against the oracle,
in both exact fp64 orders and on every engine."""

import numpy as np
import pytest

from oracle import mapper_oracle as O

pytestmark = pytest.mark.gpu

ENGINES = [1, 0]  # exact, auto (tensor-core candidates where supported)


def run(pts, rows, eps, min_pts, order=0, engine=0):
    from paper_2011_03209_b200 import DbscanParams, from_array
    from paper_2011_03209_b200.clustering import dbscan_rows

    pc = from_array(np.asarray(pts, dtype=np.float64))
    return dbscan_rows(pc, rows, DbscanParams(eps, min_pts), order=order, engine=engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_two_far_pairs(engine):  # test_clustering.py:71-75
    out = run([0.0, 0.1, 5.0, 5.1], np.arange(4), 0.2, 2, engine=engine)
    assert out.clusters == [[0, 1], [2, 3]] and out.noise == []


@pytest.mark.parametrize("engine", ENGINES)
def test_all_noise(engine):
    out = run([0.0, 10.0], np.arange(2), 1.0, 2, engine=engine)
    assert out.clusters == [] and out.noise == [0, 1]


@pytest.mark.parametrize("engine", ENGINES)
def test_eps_inclusive_and_self_counted(engine):
    out = run([0.0, 1.0], np.arange(2), 1.0, 2, engine=engine)
    assert out.clusters == [[0, 1]]


@pytest.mark.parametrize("engine", ENGINES)
def test_border_smallest_core_neighbor(engine):
    pts = [0.0, 0.4, 0.7, 1.0, 2.0, 3.0, 3.3, 3.6, 4.0]
    out = run(pts, np.arange(9), 1.0, 4, engine=engine)
    assert out.clusters == [[0, 1, 2, 3, 4], [5, 6, 7, 8]]


def test_global_row_ids_preserved():
    pts = np.zeros((31, 1))
    rows = np.array([10, 11, 20, 21, 30])
    pts[rows, 0] = [0.0, 0.1, 9.0, 9.1, 50.0]
    out = run(pts, rows, 0.5, 2, order=1)
    assert out.clusters == [[10, 11], [20, 21]] and out.noise == [30]


@pytest.mark.parametrize("seed", range(40))
@pytest.mark.parametrize("engine", ENGINES)
def test_randomized_against_oracle(seed, engine):
    rng = np.random.default_rng(7_000 + seed)
    n = int(rng.integers(1, 700))
    d = int(rng.integers(1, 70))
    pts = rng.uniform(0.0, 4.0, (n, d)) if seed % 2 else \
        O.gmm(n, d, int(rng.integers(1, 5)), 3.0, seed)
    eps = O.dist_quantile(pts, float(rng.uniform(0.02, 0.4)), seed)
    min_pts = int(rng.integers(1, 9))
    rows = np.arange(n)
    for order in (O.ORDER_SEQUENTIAL, O.ORDER_PAIRWISE):
        out = run(pts, rows, eps, min_pts, order=order, engine=engine)
        clusters, noise = O.dbscan_element(pts, rows, eps, min_pts, order)
        assert out.clusters == clusters, f"seed={seed} order={order}"
        assert out.noise == noise


@pytest.mark.parametrize("engine", ENGINES)
def test_tile_boundaries_and_many_elements(engine):
    """Elements straddling the 128-row tile size, several per launch."""
    from paper_2011_03209_b200 import DbscanParams, DistanceStrategy, cluster_all, from_array

    rng = np.random.default_rng(3)
    X = O.gmm(3000, 12, 4, 4.0, 3)
    pc = from_array(X)
    sizes = [1, 2, 127, 128, 129, 255, 256, 257, 0, 600, 1000]
    members = [np.sort(rng.choice(3000, s, replace=False)) for s in sizes]
    eps = O.dist_quantile(X, 0.1)
    strategy = DistanceStrategy(threshold=200)
    out = cluster_all(pc, members, DbscanParams(eps, 4), strategy, engine=engine)
    for k, rows in enumerate(members):
        order = O.element_order(len(rows), "precomputed", 200)
        clusters, noise = O.dbscan_element(X, rows, eps, 4, order)
        assert out[k].element_index == k
        assert out[k].clusters == clusters, k
        assert out[k].noise == noise


def test_exact_ties_follow_the_element_order():
    """The 256-D tie: cdist and numpy disagree; each order reproduces its mode."""
    import cases

    X, params = cases.tie_case()
    eps = params["eps"]
    rows = np.arange(len(X))
    pre = run(X, rows, eps, 2, order=O.ORDER_SEQUENTIAL)
    fly = run(X, rows, eps, 2, order=O.ORDER_PAIRWISE)
    assert (pre.clusters, pre.noise) == O.dbscan_element(X, rows, eps, 2, O.ORDER_SEQUENTIAL)
    assert (fly.clusters, fly.noise) == O.dbscan_element(X, rows, eps, 2, O.ORDER_PAIRWISE)
    assert pre.clusters != fly.clusters


def test_cancel_check_is_polled():
    from paper_2011_03209_b200 import DbscanParams, DistanceStrategy, cluster_all, from_array

    class Stop(Exception):
        pass

    calls = []

    def cancel():
        calls.append(1)
        raise Stop()

    pc = from_array(np.random.default_rng(0).standard_normal((50, 2)))
    with pytest.raises(Stop):
        cluster_all(pc, [np.arange(50)], DbscanParams(0.5, 3), DistanceStrategy(),
                    cancel_check=cancel)
    assert calls


@pytest.mark.parametrize("d", [5, 40, 300, 512, 600])
@pytest.mark.parametrize("engine", ENGINES)
def test_grouped_pruned_elements_against_oracle(d, engine):
    """Elements large enough for the spatial grouping and both pruning
    bounds (several seed groups over well separated blobs), for the exact
    engine at dims the tensor cores do not take (300, 512: pruning on; 600:
    pruning off) and the tensor-core engine."""
    from paper_2011_03209_b200 import DbscanParams, DistanceStrategy, cluster_all, from_array

    X = O.gmm(2600, d, 6, 6.0, 50 + d)
    eps = O.dist_quantile(X, 0.03, d)
    rng = np.random.default_rng(d)
    members = [np.sort(rng.choice(2600, s, replace=False)) for s in (2500, 1200, 400, 90)]
    cl = cluster_all(from_array(X), members, DbscanParams(eps, 4),
                     DistanceStrategy(threshold=10 ** 9), engine=engine)
    for k, m in enumerate(members):
        clusters, noise = O.dbscan_element(X, m, eps, 4, O.ORDER_SEQUENTIAL)
        assert cl[k].clusters == clusters and cl[k].noise == noise, (d, k)


@pytest.mark.parametrize("engine", ENGINES)
def test_nan_and_inf_rows(engine):
    """Non-finite coordinates: scipy's distances are NaN/inf, never <= eps, so
    those rows are noise; pruning and the tensor-core bounds must keep (not
    prune or misclassify) every tile pair touching them."""
    X = O.gmm(1500, 48, 4, 4.0, 9)
    X[[3, 700, 701]] = np.nan
    X[[40, 1200], 7] = np.inf
    X[900, 2] = -np.inf
    eps = O.dist_quantile(X[np.isfinite(X).all(axis=1)], 0.05, 9)
    rows = np.arange(1500)
    out = run(X, rows, eps, 4, order=O.ORDER_SEQUENTIAL, engine=engine)
    clusters, noise = O.dbscan_element(X, rows, eps, 4, O.ORDER_SEQUENTIAL)
    assert out.clusters == clusters and out.noise == noise


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("case", ["identical", "tiny_eps", "huge_eps", "duplicates", "one_dim_line"])
def test_degenerate_inputs(engine, case):
    """Degenerate geometry on both engines (and through the grouping/pruning
    path): zero spread, every pair in or out, duplicated rows, collinear data."""
    rng = np.random.default_rng(5)
    n, d = 900, 64
    if case == "identical":
        X, eps = np.full((n, d), 3.25), 0.5
    elif case == "tiny_eps":
        X = O.gmm(n, d, 3, 3.0, 5)
        eps = 1e-9
    elif case == "huge_eps":
        X = O.gmm(n, d, 3, 3.0, 5)
        eps = 1e6
    elif case == "duplicates":
        base = O.gmm(300, d, 3, 3.0, 5)
        X = base[rng.integers(0, 300, n)]
        eps = O.dist_quantile(base, 0.01, 5)
    else:
        t = np.sort(rng.uniform(0, 100, n))
        X = np.outer(t, np.ones(d) / np.sqrt(d))
        eps = 0.3
    rows = np.arange(n)
    for order in (O.ORDER_SEQUENTIAL, O.ORDER_PAIRWISE):
        out = run(X, rows, eps, 4, order=order, engine=engine)
        clusters, noise = O.dbscan_element(X, rows, eps, 4, order)
        assert out.clusters == clusters and out.noise == noise, (case, order)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("layout", ["blobs", "chains"])
def test_many_components_across_tiles(engine, layout):
    """Many components per 128-row tile, joined across tiles: hundreds of tight
    blobs, or long chains whose links only exist between consecutive points
    (the union-find shortcuts for symmetric diagonal tiles and single-root
    column words must not lose a join)."""
    from paper_2011_03209_b200 import DbscanParams, DistanceStrategy, cluster_all, from_array

    rng = np.random.default_rng(11 if layout == "blobs" else 12)
    d = 40
    if layout == "blobs":
        centres = rng.uniform(-50.0, 50.0, (300, d))
        X = np.repeat(centres, 8, axis=0) + 0.05 * rng.standard_normal((2400, d))
        eps = 0.6
    else:
        starts = rng.uniform(-50.0, 50.0, (12, d))
        dirs = rng.standard_normal((12, d))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        steps = np.arange(200)[:, None]
        X = np.concatenate([s + 0.4 * steps * u for s, u in zip(starts, dirs)])
        X += 0.01 * rng.standard_normal(X.shape)
        eps = 0.45
    X = X[rng.permutation(len(X))]
    members = [np.arange(len(X)), np.sort(rng.choice(len(X), 1500, replace=False))]
    for min_pts in (2, 3):
        cl = cluster_all(from_array(X), members, DbscanParams(eps, min_pts),
                         DistanceStrategy(threshold=10 ** 9), engine=engine)
        for k, m in enumerate(members):
            clusters, noise = O.dbscan_element(X, m, eps, min_pts, O.ORDER_SEQUENTIAL)
            assert len(clusters) > 10
            assert cl[k].clusters == clusters and cl[k].noise == noise, (layout, k, min_pts)
