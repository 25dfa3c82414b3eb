"""GPU, full size: the headline configuration (cfg3: 1M x 256, 40 intervals,
eps 21.3; the reference itself needs hours here).

* every node's rows and every edge equal the full-size golden
  (tests/golden/cfg3_full.npz: scipy cdist over every pair of every element,
  chunked oracle, make_golden_cfg3.py);
* the pruned build equals the build over every tile pair (pruning soundness);
* the tensor-core engine and the all-fp64 engine (parity-pinned against the
  oracle at small sizes) build identical graphs: every node's rows and every
  edge;
* lens values and cover memberships are bit-identical to the oracle's numpy
  restatement over all 1M rows;
* every element with <= 3000 rows equals the oracle's DBSCAN exactly;
* in every larger element, sampled rows obey the DBSCAN rules against exact
  fp64 distances to all rows of the element (core -> clustered; two core
  rows within eps -> same cluster; isolated -> noise; a clustered non-core
  row has a core neighbour)."""

import numpy as np
import pytest

from oracle import mapper_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg3_graphs():
    import torch

    from paper_2011_03209_b200 import DistanceStrategy, FilterSpec, MapperParams, from_array
    from paper_2011_03209_b200 import workloads
    from paper_2011_03209_b200.device import require_gpu, to_device_f64
    from paper_2011_03209_b200.pipeline import build_device

    w = workloads.CONFIGS["cfg3"]
    X = workloads.points(w)
    params = MapperParams(filters=[FilterSpec(kind="l2-norm")], n=[40], p=[0.3], eps=w.eps,
                          min_pts=w.min_pts, strategy=DistanceStrategy(threshold=10 ** 9))
    dev = require_gpu()
    Xd = to_device_f64(X, dev)
    pc = from_array(X)
    out = {}
    import os

    for engine in (2, 1, "noprune"):
        if engine == "noprune":  # tensor-core engine over EVERY tile pair
            os.environ["B200MAP_NO_PRUNE"] = "1"
        if engine == 2:  # the library checks every diagonal tile's symmetry
            os.environ["B200MAP_CHECK_SYMMETRY"] = "1"
        try:
            g = build_device(Xd, pc, params, 1 << 62, None, 2 if engine == "noprune" else engine)
        finally:
            os.environ.pop("B200MAP_NO_PRUNE", None)
            os.environ.pop("B200MAP_CHECK_SYMMETRY", None)
        out[engine] = dict(
            node_rows=g.node_rows.cpu().numpy(), node_off=g.node_off.cpu().numpy(),
            node_elem=np.asarray(g.node_elem), edges=np.asarray(g.edges),
            fv=np.asarray(g.fv_host), sizes=np.asarray(g.sizes), orders=np.asarray(g.orders),
            cover=g.cover)
        torch.cuda.synchronize()
    return X, w, out


def test_cfg3_engines_identical(cfg3_graphs):
    _, _, out = cfg3_graphs
    a, b = out[2], out[1]
    for key in ("node_rows", "node_off", "node_elem", "edges", "sizes"):
        assert np.array_equal(a[key], b[key]), key
    assert len(a["node_off"]) - 1 > 100  # a non-degenerate graph


def test_cfg3_pruning_sound_at_full_size(cfg3_graphs):
    """The pruned build equals the build that computes every tile pair of
    every element (B200MAP_NO_PRUNE=1: identity row order, 3.2e13 flop of
    distance tiles): pruning removes no eps-pair at the headline size."""
    _, _, out = cfg3_graphs
    a, b = out[2], out["noprune"]
    for key in ("node_rows", "node_off", "node_elem", "edges", "sizes"):
        assert np.array_equal(a[key], b[key]), key


def test_cfg3_equals_full_size_golden(cfg3_graphs, golden):
    """Every node's rows and every edge of the headline graph equal the
    golden made by the chunked oracle (scipy cdist itself over every pair of
    every element, union-find semantics of clustering.py:151-198; pinned to
    the reference's own goldens in test_oracle.py). make_golden_cfg3.py."""
    X, _, out = cfg3_graphs
    z = golden("cfg3_full")
    import hashlib

    assert hashlib.sha256(X.tobytes()).hexdigest() == str(z["x_sha"])
    g = out[2]
    assert np.array_equal(g["sizes"], z["sizes"])
    assert np.array_equal(g["node_off"], z["node_off"])
    assert np.array_equal(g["node_rows"], z["node_rows"].astype(np.int64))
    assert np.array_equal(g["node_elem"], z["node_elem"])
    assert np.array_equal(g["edges"].reshape(-1, 3), z["edges"])


def test_cfg3_lens_and_membership_bitwise(cfg3_graphs):
    X, w, out = cfg3_graphs
    g = out[2]
    f = O.lens(X, "l2-norm")
    assert np.array_equal(g["fv"][:, 0].view(np.int64), f.view(np.int64))
    axis = O.cover_axis(f, 40, 0.3)
    members = O.membership(f.reshape(-1, 1), [axis])
    assert np.array_equal(g["sizes"], [len(m) for m in members])


def _element_clusters(g, k):
    """Row lists of element k's nodes, in cluster order."""
    off = g["node_off"]
    ids = np.flatnonzero(g["node_elem"] == k)
    return [g["node_rows"][off[v]:off[v + 1]] for v in ids]


def _check_sampled(X, w, g, k, rows, got, rng, n_sample=16):
    """DBSCAN rules on sampled rows of element k against exact fp64 distances."""
    order = int(g["orders"][k])
    label = np.full(X.shape[0], -1, dtype=np.int64)
    for c, r in enumerate(got):
        label[np.asarray(r)] = c
    P = X[rows]

    def dist_rows(idx):
        if order == O.ORDER_SEQUENTIAL:
            return O.cdist(P[idx], P)
        return np.stack([np.sqrt(((P - P[i]) ** 2).sum(axis=1)) for i in idx])

    sample = rng.choice(rows.size, n_sample, replace=False)
    nb = dist_rows(sample) <= w.eps
    cnt = nb.sum(1)
    core = cnt >= w.min_pts
    for a, i in enumerate(sample):
        li = label[rows[i]]
        if core[a]:
            assert li >= 0, (k, i)
        if cnt[a] == 1:
            assert li < 0, (k, i)
        for b_, j in enumerate(sample):
            if core[a] and core[b_] and nb[a, j]:
                assert label[rows[j]] == li, (k, i, j)
        if li >= 0 and not core[a] and cnt[a] <= 64:
            js = np.flatnonzero(nb[a])
            assert ((dist_rows(js) <= w.eps).sum(1) >= w.min_pts).any(), (k, i)


def test_cfg3_dbscan_small_elements_exact_and_large_sampled(cfg3_graphs):
    X, w, out = cfg3_graphs
    g = out[2]
    members = O.membership(g["fv"][:, :1], [O.cover_axis(O.lens(X, "l2-norm"), 40, 0.3)])
    rng = np.random.default_rng(0)
    checked_small = checked_large = 0
    for k, rows in enumerate(members):
        rows = np.asarray(rows, dtype=np.int64)
        if rows.size == 0:
            continue
        got = [c.tolist() for c in _element_clusters(g, k)]
        if rows.size <= 3000:
            clusters, _ = O.dbscan_element(X, rows, w.eps, w.min_pts, int(g["orders"][k]))
            assert got == clusters, k
            checked_small += 1
        else:
            _check_sampled(X, w, g, k, rows, got, rng)
            checked_large += 1
    assert checked_small >= 1 and checked_large >= 10


def test_cfg5_row_block_element_sampled():
    """cfg5 (4M x 256, 10 intervals): the largest element (~1.64M rows) does
    not fit one bitmap and runs through the two-pass row-window path."""
    import torch

    from paper_2011_03209_b200 import DistanceStrategy, FilterSpec, MapperParams, from_array
    from paper_2011_03209_b200 import workloads
    from paper_2011_03209_b200.device import require_gpu, to_device_f64
    from paper_2011_03209_b200.pipeline import build_device

    w = workloads.CONFIGS["cfg5"]
    X = workloads.points(w)
    params = MapperParams(filters=[FilterSpec(kind="l2-norm")], n=[10], p=[0.3], eps=w.eps,
                          min_pts=w.min_pts, strategy=DistanceStrategy(threshold=10 ** 9))
    dev = require_gpu()
    gd = build_device(to_device_f64(X, dev), from_array(X), params, 1 << 62, None, 0)
    torch.cuda.synchronize()
    g = dict(node_rows=gd.node_rows.cpu().numpy(), node_off=gd.node_off.cpu().numpy(),
             node_elem=np.asarray(gd.node_elem), orders=np.asarray(gd.orders))
    assert int(gd.dev_stats[4]) > 0
    members = O.membership(np.asarray(gd.fv_host)[:, :1],
                           [O.cover_axis(np.asarray(gd.fv_host)[:, 0], 10, 0.3)])
    sizes = [len(m) for m in members]
    assert max(sizes) > 1_500_000
    rng = np.random.default_rng(5)
    for k in np.argsort(sizes)[::-1][:3]:
        rows = np.asarray(members[k], dtype=np.int64)
        got = [c.tolist() for c in _element_clusters(g, int(k))]
        assert sum(len(c) for c in got) <= rows.size
        _check_sampled(X, w, g, int(k), rows, got, rng, n_sample=8)


def test_cfg4_pca_grid_library_pieces():
    """cfg4 (500k x 128, 2-D PCA lens as FilterValues, 15 x 15 cover, eps 14.7)
    through the library pieces (test_nerve.py:23-30's composition): memberships
    equal the oracle's 2-D intersection, elements <= 3000 rows equal the
    oracle's DBSCAN, larger ones obey the sampled DBSCAN rules."""
    import time

    from paper_2011_03209_b200 import (DbscanParams, DistanceStrategy, FilterSpec, FilterValues,
                                       build_cover, cluster_all, from_array, membership)
    from paper_2011_03209_b200 import workloads

    w = workloads.CONFIGS["cfg4"]
    X = workloads.points(w)
    Xc = X - X.mean(axis=0)
    _, _, vt = np.linalg.svd(Xc[:20000], full_matrices=False)
    F = np.ascontiguousarray(Xc @ vt[:2].T)
    pc = from_array(X)
    fv = FilterValues(values=F.copy(), specs=[FilterSpec(kind="l2-norm")] * 2)
    t0 = time.time()
    cover = build_cover(fv, list(w.intervals), list(w.overlaps))
    members = membership(fv, cover)
    cl = cluster_all(pc, members, DbscanParams(w.eps, w.min_pts),
                     DistanceStrategy(threshold=10 ** 9))
    print(f"cfg4 library pieces: {time.time() - t0:.3f} s, "
          f"{sum(len(c.clusters) for c in cl)} clusters")
    axes = [O.cover_axis(F[:, a], w.intervals[a], w.overlaps[a]) for a in range(2)]
    want = O.membership(F, axes)
    assert [m.tolist() for m in members] == [m.tolist() for m in want]
    g = dict(orders=np.zeros(len(members), dtype=np.uint8))  # threshold 1e9: cdist order
    rng = np.random.default_rng(4)
    checked_small = checked_large = 0
    for k, rows in enumerate(members):
        rows = np.asarray(rows, dtype=np.int64)
        if rows.size == 0:
            continue
        got = [list(c) for c in cl[k].clusters]
        if rows.size <= 3000:
            clusters, noise = O.dbscan_element(X, rows, w.eps, w.min_pts, O.ORDER_SEQUENTIAL)
            assert got == clusters and list(cl[k].noise) == noise, k
            checked_small += 1
        else:
            _check_sampled(X, w, g, k, rows, got, rng, n_sample=8)
            checked_large += 1
    assert checked_small >= 5 and checked_large >= 5


def test_cfg3_default_strategy_bytes(golden):
    """A cfg3-shaped 200k x 256 cloud at the reference's DEFAULT strategy
    (threshold 20,000): 5 elements of 20-22k rows run in numpy's pairwise
    order, 35 in cdist order. The graph JSON (sha256 of every byte) equals the
    one nervemap itself produced (make_golden_cfg3d.py)."""
    import hashlib

    import cases
    from test_gpu_pipeline import graph_bytes

    z = golden("cfg3d")
    X, p = cases.cfg3_default()
    assert cases.sha(X) == str(z["x_sha"])
    got = graph_bytes(X, p)
    assert hashlib.sha256(got).hexdigest() == str(z["graph_sha"])
