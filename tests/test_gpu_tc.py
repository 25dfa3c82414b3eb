"""GPU: the tensor-core (tcgen05 kind::i8) adjacency engine decides every eps
pair exactly like the fp64 engine (and hence like the reference)."""

import numpy as np
import pytest

from oracle import mapper_oracle as O

pytestmark = pytest.mark.gpu


def labels(X, members, eps, min_pts, orders, engine):
    import torch

    from paper_2011_03209_b200 import engine as eng
    from paper_2011_03209_b200.device import require_gpu, to_device_f64

    dev = require_gpu()
    offs = np.zeros(len(members) + 1, dtype=np.int64)
    np.cumsum([len(m) for m in members], out=offs[1:])
    rows = torch.from_numpy(np.concatenate(members).astype(np.int64)).to(dev)
    lab, ncl, st = eng.cluster(to_device_f64(X, dev), rows, offs, eps, min_pts,
                               np.asarray(orders, dtype=np.uint8), engine)
    return lab.cpu().numpy(), ncl, st


@pytest.mark.parametrize("d", [32, 48, 64, 100, 128, 129, 200, 256])
@pytest.mark.parametrize("q", [0.02, 0.15])
def test_tc_equals_exact(d, q):
    rng = np.random.default_rng(d)
    X = O.gmm(2500, d, 4, 3.0, d)
    eps = O.dist_quantile(X, q, d)
    members = [np.sort(rng.choice(2500, s, replace=False)) for s in (1, 130, 700, 2100)]
    for order in (O.ORDER_SEQUENTIAL, O.ORDER_PAIRWISE):
        orders = [order] * len(members)
        a, na, _ = labels(X, members, eps, 4, orders, 1)
        b, nb, st = labels(X, members, eps, 4, orders, 2)
        assert np.array_equal(a, b) and np.array_equal(na, nb), (d, q, order)


def test_tc_matches_oracle_cfg_like():
    X = O.gmm(4000, 256, 10, 5.0, 3)
    eps = 21.3
    rows = np.arange(4000)
    lab, ncl, st = labels(X, [rows], eps, 5, [O.ORDER_SEQUENTIAL], 2)
    clusters, noise = O.dbscan_element(X, rows, eps, 5, O.ORDER_SEQUENTIAL)
    got = [rows[lab == c].tolist() for c in range(int(ncl[0]))]
    assert got == clusters
    assert rows[lab < 0].tolist() == noise
    # the recheck handles a tiny fraction of the pairs
    assert st[1] < 0.01 * st[0]


def test_tc_exact_ties():
    import cases

    X, params = cases.tie_case()
    rows = np.arange(len(X))
    for order in (O.ORDER_SEQUENTIAL, O.ORDER_PAIRWISE):
        a, _, _ = labels(X, [rows], params["eps"], 2, [order], 1)
        b, _, _ = labels(X, [rows], params["eps"], 2, [order], 2)
        assert np.array_equal(a, b)


def test_tc_large_offsets_and_nan():
    rng = np.random.default_rng(1)
    X = O.gmm(600, 64, 3, 2.0, 1) + 1e6
    X[17, 5] = np.nan
    eps = O.dist_quantile(X[np.isfinite(X).all(axis=1)], 0.1)
    rows = np.arange(600)
    a, na, _ = labels(X, [rows], eps, 3, [0], 1)
    b, nb, _ = labels(X, [rows], eps, 3, [0], 2)
    assert np.array_equal(a, b) and np.array_equal(na, nb)
    assert a[17] == -1  # NaN point is in no neighbourhood (sqrt(NaN) <= eps is False)
