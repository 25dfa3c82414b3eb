"""Probe: phases of cluster_all on cfg4's library path (dev tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03209_b200 import (DbscanParams, DistanceStrategy, FilterSpec,  # noqa: E402
                                   FilterValues, build_cover, from_array, membership, workloads)
from paper_2011_03209_b200 import clustering as C, engine as eng  # noqa: E402
from paper_2011_03209_b200.device import require_gpu, to_device_f64  # noqa: E402

w = workloads.CONFIGS["cfg4"]
X = workloads.points(w)
F = workloads.pca2_lens(X)
Xh = torch.from_numpy(X).pin_memory().numpy()
dev = require_gpu()
fv = FilterValues(values=F, specs=[FilterSpec(kind="l2-norm")] * 2)
cover = build_cover(fv, list(w.intervals), list(w.overlaps))
members = membership(fv, cover)
params = DbscanParams(w.eps, w.min_pts)
strategy = DistanceStrategy(threshold=10**9)
for rep in range(4):
    T = {}
    t = [time.perf_counter()]

    def mark(k):
        torch.cuda.current_stream(dev).synchronize()
        n = time.perf_counter()
        T[k] = (n - t[0]) * 1e3
        t[0] = n
    sizes = [int(np.asarray(r).size) for r in members]
    orders = C.element_orders(sizes, strategy, 1 << 62)
    offsets = np.zeros(len(members) + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    rows_h = np.concatenate([np.asarray(r, dtype=np.int64) for r in members])
    assert rows_h.min() >= 0 and rows_h.max() < len(X)
    mark("host_prep")
    Xd = to_device_f64(Xh, dev); mark("h2d_X")
    rows_dev = torch.from_numpy(rows_h).to(dev); mark("h2d_rows")
    labels, ncl, st = C.cluster_device(Xd, rows_dev, offsets, params, orders, None, 0); mark("dbscan")
    node_rows, node_off, _ = eng.group_nodes(rows_dev, offsets, labels, ncl); mark("group_nodes")
    lh, nrh, noh = labels.cpu().numpy(), node_rows.cpu().numpy(), node_off.cpu().numpy(); mark("d2h")
    out = C.grouped_clusterings(rows_h, offsets, lh, ncl, nrh, noh); mark("wrap")
    pc = from_array(Xh)
    t0 = time.perf_counter()
    C.cluster_all(pc, members, params, strategy, budget_bytes=1 << 62)
    torch.cuda.synchronize()
    T["cluster_all"] = (time.perf_counter() - t0) * 1e3
    print(" ".join(f"{k}={v:.2f}" for k, v in T.items()), flush=True)
