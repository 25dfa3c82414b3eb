"""CPU: host-side logic of the drop-in API (no device work)."""

import math

import numpy as np
import pytest

from oracle import mapper_oracle as O
from paper_2011_03209_b200 import (DataError, DistanceStrategy, FilterSpec, FilterValues,
                                   MapperParams, build_cover, to_canonical_json)
from paper_2011_03209_b200.clustering import (element_orders, element_uses_matrix,
                                              split_groups)


def fv_of(values):
    arr = np.asarray(values, dtype=np.float64)
    if arr.ndim == 1:
        arr = arr[:, None]
    return FilterValues(values=arr, specs=[FilterSpec(kind="l2-norm")] * arr.shape[1])


def test_cover_zero_overlap_endpoints():  # test_cover.py:21-25
    ivs = build_cover(fv_of([0.0, 1.0]), [2], [0.0]).axes[0]
    assert (ivs[0].lo, ivs[0].hi) == (0.0, 0.5)
    assert (ivs[1].lo, ivs[1].hi) == (0.5, 1.0)


def test_cover_degenerate_axis():  # test_cover.py:77-84
    with pytest.warns(UserWarning, match="constant filter"):
        cover = build_cover(fv_of([4.0, 4.0, 4.0]), [5], [0.3])
    assert cover.n == [1]
    assert (cover.axes[0][0].lo, cover.axes[0][0].hi) == (3.5, 4.5)


def test_cover_invalid():
    fv = fv_of([0.0, 1.0])
    for n, p in (([0], [0.3]), ([3], [0.96]), ([3, 3], [0.3])):
        with pytest.raises(DataError):
            build_cover(fv, n, p)


@pytest.mark.parametrize("seed", range(20))
def test_cover_endpoints_match_oracle(seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(50) * rng.uniform(0.01, 1000)
    n = int(rng.integers(1, 40))
    p = float(rng.uniform(0, 0.95))
    ivs = build_cover(fv_of(v), [n], [p]).axes[0]
    assert [(iv.lo, iv.hi) for iv in ivs] == O.cover_axis(v, n, p)


def test_2d_element_keys():  # test_cover.py:97-108
    vals = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    fv = FilterValues(values=vals, specs=[FilterSpec(kind="l2-norm")] * 2)
    cover = build_cover(fv, [2, 3], [0.0, 0.0])
    assert cover.n_elements == 6
    assert cover.element_key(0) == [0, 0]
    assert cover.element_key(2) == [0, 2]
    assert cover.element_key(3) == [1, 0]


def test_strategy_and_params_validation():
    with pytest.raises(DataError):
        DistanceStrategy(mode="gpu")  # test_clustering.py:144: GPU is not a strategy mode
    with pytest.raises(DataError):
        DistanceStrategy(threshold=0)
    with pytest.raises(DataError):
        MapperParams(filters=[], n=[], p=[], eps=1.0)
    with pytest.raises(DataError):
        MapperParams(filters=[FilterSpec(kind="l2-norm")], n=[3], p=[0.3], eps=0.0)
    with pytest.raises(DataError):
        MapperParams(filters=[FilterSpec(kind="l2-norm")], n=[3], p=[0.3], eps=1.0, norm="zz")


def test_manifest_is_mode_free():
    a = MapperParams(filters=[FilterSpec(kind="l2-norm")], n=[3], p=[0.3], eps=1.0,
                     strategy=DistanceStrategy(mode="on-the-fly", threshold=7))
    assert a.manifest()["strategy"] == {"threshold": 7}
    assert to_canonical_json(a.manifest()) == (
        b'{"eps":1,"filters":[{"kind":"l2-norm"}],"min_pts":5,"n":[3],"norm":"none",'
        b'"p":[0.3],"strategy":{"threshold":7}}')


def test_filter_spec_json():
    s = FilterSpec.from_json_obj({"kind": "eccentricity", "p": "inf"})
    assert s.p == math.inf and s.to_json_obj() == {"kind": "eccentricity", "p": "inf"}
    with pytest.raises(DataError):
        FilterSpec.from_json_obj({"kind": "column"})
    with pytest.raises(DataError):
        FilterSpec.from_json_obj({"kind": "l2-norm", "bogus": 1})


def test_order_choice_mirrors_reference():
    st = DistanceStrategy(threshold=100)
    assert element_uses_matrix(100, st, 10**9)
    assert not element_uses_matrix(101, st, 10**9)
    assert not element_uses_matrix(100, st, 100 * 100 * 8 - 1)
    assert not element_uses_matrix(5, DistanceStrategy(mode="on-the-fly"), 10**9)
    o = element_orders([5, 500], st, 10**9)
    assert o.tolist() == [0, 1]
    for n in (0, 5, 100, 101, 20_000, 20_001):
        assert int(element_uses_matrix(n, DistanceStrategy(), 8 << 30)) == \
            int(O.element_order(n) == O.ORDER_SEQUENTIAL)


def test_split_groups_cover_all_elements():
    offs = np.cumsum([0, 5, 0, 7, 3, 9, 0])
    groups = split_groups(offs, limit=10)
    assert groups[0][0] == 0 and groups[-1][1] == len(offs) - 1
    for (a, b), (c, d) in zip(groups, groups[1:]):
        assert b == c


def test_canonical_float_format():
    assert to_canonical_json([1e-5, -0.0, 0.1, 123456789012.0, 2.5]) == \
        b"[1e-05,0,0.1,1.23456789e+11,2.5]"
    with pytest.raises(DataError):
        to_canonical_json([float("nan")])


def test_split_groups_pair_work_limit():
    """With a cancel_check, groups are also bounded by sum n_k^2 (cfg5-scale
    builds poll several times); an element above the limit is alone."""
    sizes = [100, 5, 5, 300, 1, 1, 200]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    groups = split_groups(offs, limit=10 ** 9, pair_limit=100 ** 2 + 60)
    assert [k for a, b in groups for k in range(a, b)] == list(range(len(sizes)))
    for a, b in groups:
        work = sum(s * s for s in sizes[a:b])
        assert b - a == 1 or work <= 100 ** 2 + 60
    assert split_groups(offs, limit=10 ** 9) == [(0, len(sizes))]


def test_pullback_clustering_lazy_lists():
    """cluster_all's results hold flat arrays until clusters/noise are read;
    then they are the reference's plain lists (equality, repr, pickle, copy),
    and flat_clusters stops trusting them once a caller edits a list."""
    import copy
    import pickle

    from paper_2011_03209_b200.clustering import PullbackClustering, flat_clusters

    flat = np.array([3, 7, 9, 1, 2], dtype=np.int64)
    sizes = np.array([3, 2], dtype=np.int64)
    noise = np.array([4, 11], dtype=np.int64)
    want = PullbackClustering(5, [[3, 7, 9], [1, 2]], [4, 11])

    p = PullbackClustering._from_flat(5, flat, sizes, noise)
    fr, fs = flat_clusters(p)  # no lists built yet
    assert fr is flat and fs is sizes and "clusters" not in p.__dict__
    q = pickle.loads(pickle.dumps(p))
    r = copy.deepcopy(p)
    assert p == want and q == want and r == want and repr(p) == repr(want)
    assert all(type(v) is int for c in p.clusters for v in c) and type(p.noise) is list
    fr, fs = flat_clusters(p)  # lists built and untouched: still the flat arrays
    assert fr.tolist() == [3, 7, 9, 1, 2] and fs.tolist() == [3, 2]
    p.clusters[0].append(12)
    assert flat_clusters(p) is None
    with pytest.raises(AttributeError):
        p.missing  # noqa: B018
    assert flat_clusters(want) is None  # a caller-built result has no flat copy
