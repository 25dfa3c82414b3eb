"""Small builds for compute-sanitizer (memcheck / racecheck / synccheck):
cfg1 through compute_mapper (exact engine, d = 3) and a d = 64 cloud on the
tensor-core engine (tcgen05 + TMA + mbarrier pipeline, recheck, union-find).

    compute-sanitizer --tool memcheck python scripts/probe_sanitize.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import numpy as np  # noqa: E402

import cases  # noqa: E402
from oracle import mapper_oracle as O  # noqa: E402
from paper_2011_03209_b200 import (DistanceStrategy, FilterSpec, MapperParams,  # noqa: E402
                                   compute_mapper, from_array)

X, p = cases.cfg1()
params = MapperParams(filters=[FilterSpec(kind="column", column="x0")], n=[10], p=[0.3],
                      eps=0.5, min_pts=5)
run = compute_mapper(from_array(X), params)
z = np.load(os.path.join(ROOT, "tests", "golden", "cfg1.npz"))
assert run.graph_bytes == z["graph"].tobytes(), "cfg1 bytes differ"
print("cfg1 ok", run.graph.n_nodes)

X = O.gmm(3000, 64, 4, 4.0, 11)
eps = O.dist_quantile(X, 0.05)
params = MapperParams(filters=[FilterSpec(kind="l2-norm")], n=[3], p=[0.3], eps=eps, min_pts=4,
                      strategy=DistanceStrategy(threshold=10 ** 9))
run = compute_mapper(from_array(X), params, engine=2)
want = O.mapper_graph(X, [("l2-norm", 0)], [3], [0.3], eps, 4, threshold=10 ** 9)
assert [n.rows for n in run.graph.nodes] == want["node_rows"], "tc nodes differ"
print("tc d=64 ok", run.graph.n_nodes)
