"""Probe: time each library piece of cfg4's reference-facing path
(build_cover -> membership -> cluster_all -> build_graph -> graph_to_json)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03209_b200 import (DbscanParams, DistanceStrategy, FilterSpec,  # noqa: E402
                                   FilterValues, build_cover, build_graph, cluster_all,
                                   from_array, graph_to_json, membership, workloads)

w = workloads.CONFIGS["cfg4"]
X = workloads.points(w)
F = workloads.pca2_lens(X)
Xh = torch.from_numpy(X).pin_memory().numpy()
Fh = torch.from_numpy(F).pin_memory().numpy()
for it in range(3):
    t = [time.perf_counter()]
    pc = from_array(Xh)
    fv = FilterValues(values=Fh, specs=[FilterSpec(kind="l2-norm")] * 2)
    cover = build_cover(fv, list(w.intervals), list(w.overlaps)); t.append(time.perf_counter())
    members = membership(fv, cover); t.append(time.perf_counter())
    cl = cluster_all(pc, members, DbscanParams(w.eps, w.min_pts), DistanceStrategy(threshold=10**9),
                     budget_bytes=1 << 62); t.append(time.perf_counter())
    g = build_graph(cl, pc, fv, cover, manifest={}); t.append(time.perf_counter())
    b = graph_to_json(g); t.append(time.perf_counter())
    names = ["cover", "membership", "cluster_all", "build_graph", "json"]
    print(" ".join(f"{n} {1e3 * (t[i + 1] - t[i]):.1f}" for i, n in enumerate(names)),
          f"total {1e3 * (t[-1] - t[0]):.1f} ms", flush=True)
