"""GPU end-to-end parity: compute_mapper graph bytes are byte-identical to the
reference's (golden fixtures made by running nervemap; make_golden.py)."""

import numpy as np
import pytest

import cases
from oracle import mapper_oracle as O

pytestmark = pytest.mark.gpu


def params_of(p):
    from paper_2011_03209_b200 import DistanceStrategy, FilterSpec, MapperParams

    return MapperParams(filters=[FilterSpec.from_json_obj(f) for f in p["filters"]], n=p["n"],
                        p=p["p"], eps=p["eps"], min_pts=p["min_pts"], norm=p["norm"],
                        strategy=DistanceStrategy(mode=p["mode"], threshold=p["threshold"]))


def graph_bytes(X, p, engine=0):
    from paper_2011_03209_b200 import DataError, compute_mapper, from_array

    try:
        return compute_mapper(from_array(X), params_of(p), engine=engine).graph_bytes
    except DataError as e:
        return ("DataError: " + str(e)).encode()


@pytest.mark.parametrize("engine", [1, 0])
def test_cfg1_bytes(golden, engine):
    z = golden("cfg1")
    X, p = cases.cfg1()
    assert cases.sha(X) == str(z["x_sha"])
    assert graph_bytes(X, p, engine) == z["graph"].tobytes()


@pytest.mark.parametrize("engine", [1, 0])
def test_cfg2_bytes(golden, engine):
    z = golden("cfg2")
    X, p = cases.cfg2()
    assert cases.sha(X) == str(z["x_sha"])
    assert graph_bytes(X, p, engine) == z["graph"].tobytes()


@pytest.mark.parametrize("seed", range(cases.N_INSTANCES))
def test_instances_bytes(golden, seed):
    z = golden("instances")
    X, p = cases.instance(seed)
    assert cases.sha(X) == str(z["x_sha"][seed])
    assert graph_bytes(X, p) == z[f"g{seed}"].tobytes()


def test_tie_bytes_both_modes(golden):
    z = golden("tie")
    X, p = cases.tie_case()
    assert graph_bytes(X, dict(p, mode="precomputed")) == z["pre"].tobytes()
    assert graph_bytes(X, dict(p, mode="on-the-fly")) == z["fly"].tobytes()


def test_pca2d_library_pieces(golden):
    """Config-4 shape: a 2-D lens supplied as FilterValues (test_nerve.py:23-30)."""
    from paper_2011_03209_b200 import (DbscanParams, DistanceStrategy, FilterSpec, FilterValues,
                                       build_cover, build_graph, cluster_all, from_array,
                                       graph_to_json, membership)

    z = golden("pca2d")
    X, _, q = cases.pca2d_case()
    assert cases.sha(X) == str(z["x_sha"])
    F = z["F"]
    pc = from_array(X)
    fv = FilterValues(values=F.copy(), specs=[FilterSpec(kind="l2-norm")] * 2)
    cover = build_cover(fv, q["n"], q["p"])
    members = membership(fv, cover)
    assert [m.size for m in members] == z["sizes"].tolist()
    cl = cluster_all(pc, members, DbscanParams(q["eps"], q["min_pts"]), DistanceStrategy())
    g = build_graph(cl, pc, fv, cover, manifest={"test": True})
    assert graph_to_json(g) == z["graph"].tobytes()
    # build_graph's flat fast path (lists made by cluster_all) and the generic
    # path (caller-built lists; one edited in place) give the same bytes
    from paper_2011_03209_b200 import PullbackClustering
    from paper_2011_03209_b200.clustering import flat_clusters

    assert all(flat_clusters(c) is not None for c in cl)
    cl2 = [PullbackClustering(c.element_index, [list(m) for m in c.clusters], list(c.noise))
           for c in cl]
    assert cl2 == cl
    assert all(flat_clusters(c) is None for c in cl2)
    assert graph_to_json(build_graph(cl2, pc, fv, cover, manifest={"test": True})) == \
        z["graph"].tobytes()
    k = next(i for i, c in enumerate(cl) if c.clusters)
    cl[k].clusters[0].append(cl[k].clusters[0].pop())  # same length, same content
    cl[k].clusters.append([])  # resized: the generic path for element k
    assert flat_clusters(cl[k]) is None
    cl[k].clusters.pop()


def test_modes_and_thresholds_identical_when_no_ties():
    """Mirror of test_clustering.py:163-190 on a snowman-like cloud."""
    from paper_2011_03209_b200 import (ClusterRunStats, DbscanParams, DistanceStrategy,
                                       FilterSpec, FilterValues, build_cover, cluster_all,
                                       from_array, membership)

    rng = np.random.default_rng(7)
    tb, th = rng.uniform(0, 2 * np.pi, 400), rng.uniform(0, 2 * np.pi, 240)
    pts = np.vstack([np.column_stack([np.cos(tb), np.sin(tb)]),
                     np.column_stack([0.5 * np.cos(th), 1.3 + 0.5 * np.sin(th)])])
    pc = from_array(pts, names=["x", "y"])
    fv = FilterValues(values=pts[:, 1:2].copy(), specs=[FilterSpec(kind="column", column="y")])
    members = membership(fv, build_cover(fv, [6], [0.3]))
    prm = DbscanParams(0.35, 3)
    base = cluster_all(pc, members, prm, DistanceStrategy())
    assert len(base[0].clusters) == 1 and len(base[1].clusters) == 2
    for strat in (DistanceStrategy(mode="on-the-fly"), DistanceStrategy(threshold=10)):
        st = ClusterRunStats()
        other = cluster_all(pc, members, prm, strat, stats_out=st, threads=4)
        assert [(r.clusters, r.noise) for r in other] == [(r.clusters, r.noise) for r in base]
    st = ClusterRunStats()
    cluster_all(pc, members, prm, DistanceStrategy(threshold=10), stats_out=st)
    assert st.matrix_elements == 0 and st.fallback_elements > 0


def test_nerve_edges_sparse_path_matches_oracle():
    """More than 4096 nodes exercises the sort-based edge path of K7."""
    import torch

    from paper_2011_03209_b200 import engine
    from paper_2011_03209_b200.device import require_gpu

    dev = require_gpu()
    rng = np.random.default_rng(5)
    n_points, n_nodes = 20_000, 5000
    node_rows = [np.sort(rng.choice(n_points, int(rng.integers(1, 12)), replace=False))
                 for _ in range(n_nodes)]
    off = np.zeros(n_nodes + 1, dtype=np.int64)
    np.cumsum([len(r) for r in node_rows], out=off[1:])
    flat = np.concatenate(node_rows)
    edges = engine.nerve_edges(torch.from_numpy(flat).to(dev), torch.from_numpy(off).to(dev),
                               n_nodes, n_points)
    want = O.nerve_edges_fast([r.tolist() for r in node_rows], n_points)
    assert [tuple(e) for e in edges.tolist()] == want


@pytest.mark.parametrize("max_nodes_per_point", [2, 4, 8, 9, 30])
def test_nerve_edges_dense_slots_and_overflow(max_nodes_per_point):
    """Dense path (<= 4096 nodes): points in <= 8 nodes take the sort-free
    slot path; a point in more nodes sends the call down the sorting path.
    Both equal the oracle's nerve edges."""
    import torch

    from paper_2011_03209_b200 import engine
    from paper_2011_03209_b200.device import require_gpu

    dev = require_gpu()
    rng = np.random.default_rng(max_nodes_per_point)
    n_points, n_nodes = 30_000, 300
    member = [[] for _ in range(n_nodes)]
    for p in range(n_points):
        k = int(rng.integers(1, max_nodes_per_point + 1)) if p % 7 == 0 else int(rng.integers(1, 3))
        for v in rng.choice(n_nodes, min(k, max_nodes_per_point), replace=False):
            member[v].append(p)
    node_rows = [np.array(sorted(m), dtype=np.int64) for m in member if m]
    off = np.zeros(len(node_rows) + 1, dtype=np.int64)
    np.cumsum([len(r) for r in node_rows], out=off[1:])
    flat = np.concatenate(node_rows)
    edges = engine.nerve_edges(torch.from_numpy(flat).to(dev), torch.from_numpy(off).to(dev),
                               len(node_rows), n_points)
    want = O.nerve_edges_fast([r.tolist() for r in node_rows], n_points)
    assert [tuple(e) for e in edges.tolist()] == want
