"""cfg4 through the library pieces, timed per stage (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2011_03209_b200 import (DbscanParams, DistanceStrategy, FilterSpec, FilterValues,
                                   build_cover, build_graph, cluster_all, from_array, membership)
from paper_2011_03209_b200 import workloads
w = workloads.CONFIGS["cfg4"]
X = workloads.points(w)
Xc = X - X.mean(axis=0)
_, _, vt = np.linalg.svd(Xc[:20000], full_matrices=False)
F = np.ascontiguousarray(Xc @ vt[:2].T)
pc = from_array(X)
fv = FilterValues(values=F.copy(), specs=[FilterSpec(kind="l2-norm")] * 2)
for it in range(3):
    t = [time.time()]
    cover = build_cover(fv, list(w.intervals), list(w.overlaps)); t.append(time.time())
    members = membership(fv, cover); t.append(time.time())
    cl = cluster_all(pc, members, DbscanParams(w.eps, w.min_pts), DistanceStrategy(threshold=10 ** 9)); t.append(time.time())
    g = build_graph(cl, pc, fv, cover, manifest={}); t.append(time.time())
    print(it, "cover %.3f membership %.3f cluster_all %.3f build_graph %.3f" % tuple(np.diff(t)),
          "nodes", g.n_nodes, "edges", len(g.edges), flush=True)
