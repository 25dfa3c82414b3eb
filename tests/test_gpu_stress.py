"""GPU parity under stress: planted near-eps decisions in 256-D, data whose
squared differences underflow, and the diagonal-tile symmetry invariant.

* near_eps: 3,200 planted links whose cdist length is within +-2 ulp of eps
  (tests/golden/near_eps.npz, made by running nervemap in both strategy
  modes). Both summation orders, both engines, pruning on: the graph bytes'
  sha256 equals the reference's.
* tiny scale: data and eps scaled by 1e-160, so (x_i - x_j)^2 is subnormal
  and the reference's distances carry large relative error; the engine must
  reproduce them bit for bit (no pruning, every tensor-core decision
  rechecked; dbscan.cu eps_in_model).
* B200MAP_CHECK_SYMMETRY=1 makes the library check every diagonal tile
  bitmap against its transpose (the diagonal union-find pass relies on it)."""

import hashlib

import numpy as np
import pytest

import cases
from oracle import mapper_oracle as O
from test_gpu_pipeline import graph_bytes

pytestmark = pytest.mark.gpu


@pytest.fixture
def symmetry_check(monkeypatch):
    monkeypatch.setenv("B200MAP_CHECK_SYMMETRY", "1")


@pytest.mark.parametrize("engine", [2, 1])
@pytest.mark.parametrize("mode,key", [("precomputed", "pre"), ("on-the-fly", "fly")])
def test_near_eps_links_bytes(golden, symmetry_check, engine, mode, key):
    z = golden("near_eps")
    X, p = cases.near_eps_case()
    assert cases.sha(X) == str(z["x_sha"])
    got = graph_bytes(X, dict(p, mode=mode), engine)
    assert hashlib.sha256(got).hexdigest() == str(z[f"{key}_sha"])


@pytest.mark.parametrize("engine", [2, 1])
def test_near_eps_links_pruning_off_equal(golden, monkeypatch, engine):
    """Pruning never changes a near-eps decision."""
    z = golden("near_eps")
    X, p = cases.near_eps_case()
    monkeypatch.setenv("B200MAP_NO_PRUNE", "1")
    got = graph_bytes(X, dict(p, mode="precomputed"), engine)
    assert hashlib.sha256(got).hexdigest() == str(z["pre_sha"])


@pytest.mark.parametrize("engine", [2, 1])
@pytest.mark.parametrize("order", [O.ORDER_SEQUENTIAL, O.ORDER_PAIRWISE])
def test_subnormal_scale_matches_oracle(symmetry_check, engine, order):
    from paper_2011_03209_b200 import DbscanParams, dbscan_rows, from_array

    X = O.gmm(3000, 64, 4, 4.0, 21) * 1e-160
    eps = O.dist_quantile(X, 0.05)
    assert eps < 1e-140
    assert ((X[0] - X[1]) ** 2 < np.finfo(np.float64).tiny).all()  # subnormal squares
    rows = np.arange(3000)
    got = dbscan_rows(from_array(X), rows, DbscanParams(eps, 4), order=order, engine=engine)
    want, noise = O.dbscan_element(X, rows, eps, 4, order)
    assert got.clusters == want and got.noise == noise


@pytest.mark.parametrize("engine", [2, 1])
def test_random_instances_symmetry(symmetry_check, engine):
    """Diagonal tiles are symmetric on the randomized 256-D instances (the
    library raises InternalError otherwise)."""
    from paper_2011_03209_b200 import DbscanParams, dbscan_rows, from_array

    for seed in range(6):
        X = O.gmm(2500, 256, 6, 3.0, 300 + seed)
        eps = O.dist_quantile(X, 0.02 + 0.05 * seed)
        got = dbscan_rows(from_array(X), np.arange(len(X)), DbscanParams(eps, 5),
                          order=seed % 2, engine=engine)
        want, noise = O.dbscan_element(X, np.arange(len(X)), eps, 5, seed % 2)
        assert got.clusters == want and got.noise == noise, seed
