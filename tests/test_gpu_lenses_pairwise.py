"""GPU: eccentricity and density lenses (filters.py:103-150) against the
reference's own values (tests/golden/plens.npz, produced by running nervemap):
p in {1, 2, inf} bit-exact, density and p = 3 within the ulp-level exp/pow
differences (relative 1e-13), both for targets = all points (900 rows) and
for the seed-1729 subsample of 50,000 targets (52,000 rows, default
bandwidth from the 1000-point subsample)."""

import os

import numpy as np
import pytest

import cases

pytestmark = pytest.mark.gpu

SPECS = {"ecc1": dict(kind="eccentricity"), "ecc2": dict(kind="eccentricity", p=2.0),
         "ecc3": dict(kind="eccentricity", p=3.0),
         "eccinf": dict(kind="eccentricity", p=float("inf")),
         "dens": dict(kind="density"), "dens17": dict(kind="density", bandwidth=1.7)}
EXACT = {"ecc1", "ecc2", "eccinf"}


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "plens.npz"))


@pytest.mark.parametrize("tag,n,d,seed,names", [
    ("small", 900, 5, 11, list(SPECS)),
    ("big", 52_000, 3, 12, ["ecc1", "eccinf", "dens"]),
])
def test_pairwise_lenses_match_reference(golden, tag, n, d, seed, names):
    from paper_2011_03209_b200 import FilterSpec, evaluate, from_array

    X = cases.gmm(n, d, 4, 3.0, seed)
    assert cases.sha(X) == str(golden[f"{tag}_sha"])
    pc = from_array(X)
    for name in names:
        got = evaluate(pc, FilterSpec(**SPECS[name]))
        want = golden[f"{tag}_{name}"]
        if name in EXACT:
            assert np.array_equal(got, want), name
        else:
            np.testing.assert_allclose(got, want, rtol=1e-13, atol=0, err_msg=name)


def test_pairwise_lens_pipeline_end_to_end():
    """compute_mapper with an eccentricity lens builds the same graph as the
    oracle pipeline fed with the oracle's lens values."""
    from oracle import mapper_oracle as O
    from paper_2011_03209_b200 import (DistanceStrategy, FilterSpec, MapperParams, compute_mapper,
                                       from_array)

    X = cases.gmm(3000, 8, 5, 3.0, 21)
    eps = O.dist_quantile(X, 0.03, 1)
    params = MapperParams(filters=[FilterSpec(kind="eccentricity")], n=[8], p=[0.3], eps=eps,
                          min_pts=4, strategy=DistanceStrategy(threshold=10 ** 9))
    run = compute_mapper(from_array(X), params)
    f = O.pairwise_lens(X, "eccentricity")
    assert np.array_equal(run.fv.values[:, 0], f)
    members = O.membership(f.reshape(-1, 1), [O.cover_axis(f, 8, 0.3)])
    want = []
    for k, rows in enumerate(members):
        clusters, _ = O.dbscan_element(X, rows, eps, 4, O.ORDER_SEQUENTIAL)
        want += clusters
    assert [n.rows for n in run.graph.nodes] == want
