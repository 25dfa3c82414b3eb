"""Generate the full-size headline golden (cfg3: 1M x 256, l2-norm lens,
40 intervals, 30% overlap, eps 21.3, min_pts 5; strategy threshold >= max n_k,
so every element is clustered in the reference's cdist order — the setting
bench.py times).

No dense reference run is possible here (the largest element's matrix is
142 GB), so the DBSCAN of every element is evaluated by the chunked oracle
(oracle/chunked.py): scipy cdist itself (clustering.py:113) over row blocks of
the upper triangle, eps-pairs kept, union-find semantics of
clustering.py:151-198. The chunked oracle is pinned to the dense oracle and to
the reference's own golden graphs in tests/test_oracle.py.

    python tests/golden/make_golden_cfg3.py [--workers 7] [--config cfg3]

Writes tests/golden/<config>_full.npz: the node rows (int32, concatenated in
node order), node offsets, node elements, the edge list and the element sizes,
plus a sha256 of X. A run takes ~1 h on 8 cores.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import chunked as C  # noqa: E402
from oracle import mapper_oracle as O  # noqa: E402
from paper_2011_03209_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=7)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--block", type=int, default=1024)
    args = ap.parse_args()
    w = workloads.CONFIGS[args.config]
    X = workloads.points(w)
    sha = hashlib.sha256(X.tobytes()).hexdigest()
    F = np.column_stack([O.lens(X, k, int(c[1:]) if c else 0) for k, c in w.lens])
    axes = [O.cover_axis(F[:, a], w.intervals[a], w.overlaps[a]) for a in range(F.shape[1])]
    members = O.membership(F, axes)
    sizes = np.array([m.size for m in members], dtype=np.int64)
    print(f"{args.config}: {len(members)} elements, max {sizes.max()}, "
          f"sum n^2 {float((sizes.astype(float) ** 2).sum()):.3e}", flush=True)
    node_rows, node_elem = [], []
    t0 = time.time()
    results = {}
    for k in range(len(members)):
        t = time.time()
        results[k] = C.dbscan_element(X, members[k], w.eps, w.min_pts, O.ORDER_SEQUENTIAL,
                                      block=args.block, workers=args.workers)
        print(f"element {k}: {sizes[k]} rows, {len(results[k][0])} clusters, "
              f"{len(results[k][1])} noise, {time.time() - t:.1f}s (total {time.time() - t0:.0f}s)",
              flush=True)
    for k in range(len(members)):
        for c in results[k][0]:
            node_rows.append(c)
            node_elem.append(k)
    edges = O.nerve_edges_fast(node_rows, X.shape[0])
    off = np.zeros(len(node_rows) + 1, dtype=np.int64)
    np.cumsum([len(r) for r in node_rows], out=off[1:])
    flat = (np.concatenate([np.asarray(r, dtype=np.int32) for r in node_rows])
            if node_rows else np.zeros(0, np.int32))
    path = os.path.join(HERE, f"{args.config}_full.npz")
    np.savez_compressed(path, x_sha=np.array(sha), sizes=sizes,
                        node_elem=np.asarray(node_elem, dtype=np.int32), node_off=off,
                        node_rows=flat, edges=np.asarray(edges, dtype=np.int64).reshape(-1, 3),
                        eps=np.array(w.eps), min_pts=np.array(w.min_pts))
    print(f"wrote {path} ({os.path.getsize(path)} bytes): {len(node_rows)} nodes, "
          f"{len(edges)} edges, {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()
