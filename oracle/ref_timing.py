"""ORACLE (TEST INFRASTRUCTURE ONLY) — timing of the reference's CPU path for
bench.py's CPU baseline and `--impl reference` arm. Nothing here is on the
product path; bench.py runs it on the host cores only.

The reference (nervemap, pure numpy/scipy; /root/reference does not exist on
the GPU box) is timed through its step-for-step port in mapper_oracle
(lens, cover, membership, dbscan_bfs, nerve, payload), scheduled like
clustering.py:238-316 (fork pool, elements submitted in element order, at
most 2 x threads in flight).

Two measurements:
* full_build(): one whole Mapper build, end to end, on `workers` processes —
  feasible for cfg1/cfg2 (tens of seconds);
* element_rate_sample(): for workloads the reference cannot finish in a
  bench run (cfg3: ~1-2 h on a many-core host), EVERY cover element is
  sampled — r evenly spaced rows of each element run the reference's per-row
  work (the cdist row against the whole element, the count_nonzero scan, the
  BFS neighbour query and its per-neighbour Python loop) — and each element's
  time is its sampled per-row time x n_k. The per-element times are then
  scheduled like the reference's pool (schedule_makespan). The per-row cost
  of an element is uniform across its rows, so the extrapolation is linear
  in rows, never in n_k^2.
"""

from __future__ import annotations

import multiprocessing as mp
import time
from concurrent.futures import FIRST_COMPLETED, ProcessPoolExecutor, wait

import numpy as np
from scipy.spatial.distance import cdist

from . import mapper_oracle as O

_CTX: dict = {}


def _init(ctx):
    _CTX.clear()
    _CTX.update(ctx)


def _pool(workers):
    return ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork"),
                               initializer=_init, initargs=(dict(_CTX),))


# ---------------------------------------------------------------------------
# whole build (cluster_all's scheduler: clustering.py:281-315)
# ---------------------------------------------------------------------------
def _run_element(k):
    c = _CTX
    t = time.perf_counter()
    res = O.dbscan_element_bfs(c["X"], c["members"][k], c["eps"], c["min_pts"], c["orders"][k])
    return k, res, time.perf_counter() - t


def cluster_all_reference_schedule(X, members, eps, min_pts, orders, workers):
    """Per-element results and single-worker seconds, run like the reference's
    pool: submission in element order with <= 2 x workers in flight."""
    _CTX.update(X=X, members=members, eps=eps, min_pts=min_pts, orders=orders)
    out = [None] * len(members)
    secs = [0.0] * len(members)
    if workers <= 1 or len(members) <= 1:
        for k in range(len(members)):
            _, out[k], secs[k] = _run_element(k)
        return out, secs
    pending = list(range(len(members)))
    with _pool(workers) as pool:
        in_flight = set()
        while pending or in_flight:
            while pending and len(in_flight) < 2 * workers:
                in_flight.add(pool.submit(_run_element, pending.pop(0)))
            done, in_flight = wait(in_flight, return_when=FIRST_COMPLETED)
            for f in done:
                k, res, s = f.result()
                out[k], secs[k] = res, s
    return out, secs


def full_build(X, lenses, n, p, eps, min_pts, threshold=O.DEFAULT_PRECOMPUTE_THRESHOLD,
               budget=O.DEFAULT_MEM_BUDGET_BYTES, workers=1) -> dict:
    """One reference Mapper build (pipeline.py:81-110 minus the JSON writer),
    timed stage by stage on `workers` processes."""
    t0 = time.perf_counter()
    F = np.column_stack([O.lens(X, k, c) for k, c in lenses])
    axes = [O.cover_axis(F[:, a], n[a], p[a]) for a in range(F.shape[1])]
    members = O.membership(F, axes)
    t1 = time.perf_counter()
    orders = [O.element_order(len(r), "precomputed", threshold, budget) for r in members]
    results, secs = cluster_all_reference_schedule(X, members, eps, min_pts, orders, workers)
    t2 = time.perf_counter()
    node_rows = [c for clusters, _ in results for c in clusters]
    edges = O.nerve_edges_fast(node_rows, X.shape[0])
    O.node_payload(X, F, node_rows)
    t3 = time.perf_counter()
    return {"seconds": t3 - t0, "lens_cover_s": t1 - t0, "cluster_s": t2 - t1,
            "nerve_payload_s": t3 - t2, "single_worker_cluster_s": float(sum(secs)),
            "workers": workers, "nodes": len(node_rows), "edges": len(edges)}


# ---------------------------------------------------------------------------
# sampled per-element rates (workloads beyond a bench run)
# ---------------------------------------------------------------------------
def _sample_rows(k, idx):
    """Seconds of the reference's per-row work for rows idx of element k."""
    c = _CTX
    rows = c["members"][k]
    t = time.perf_counter()
    P = c["X"][rows]
    eps, min_pts = c["eps"], c["min_pts"]
    if c["orders"][k] == O.ORDER_SEQUENTIAL:
        D = cdist(P[idx], P)                           # clustering.py:113
        cnt = np.count_nonzero(D <= eps, axis=1)       # :123-124
        nbr_rows = [np.flatnonzero(D[a] <= eps) for a in range(len(idx))]  # :126-127
    else:
        def row(i):                                    # clustering.py:137-139
            diff = P - P[i]
            return np.sqrt((diff * diff).sum(axis=1))
        cnt = np.array([np.count_nonzero(row(i) <= eps) for i in idx])
        nbr_rows = [np.flatnonzero(row(i) <= eps) for i in idx]
    # the BFS inner loop (clustering.py:177-181) visits every neighbour of
    # every visited point; in the dense elements nearly every point is core
    # and already labelled when revisited
    core = np.ones(len(rows), dtype=bool)
    labels = np.zeros(len(rows), dtype=np.int64)
    hits = 0
    for nb in nbr_rows:
        for j in nb:
            if core[j] and labels[j] < 0:
                hits += 1
    _ = (cnt >= min_pts).sum() + hits
    return k, len(idx), time.perf_counter() - t


def element_rate_sample(X, members, eps, min_pts, orders, rows_per_element, workers,
                        seed=0, chunk=256) -> dict:
    """Per-element seconds per row from r evenly spaced rows of every element
    (r = min(n_k, rows_per_element)), measured on `workers` busy processes."""
    _CTX.update(X=X, members=members, eps=eps, min_pts=min_pts, orders=orders)
    rng = np.random.default_rng(seed)
    tasks = []
    for k, m in enumerate(members):
        nk = len(m)
        if nk == 0:
            continue
        r = min(nk, rows_per_element)
        off = int(rng.integers(0, max(nk // r, 1)))
        idx = np.minimum((np.arange(r) * (nk / r)).astype(np.int64) + off, nk - 1)
        for a in range(0, r, chunk):
            tasks.append((k, idx[a:a + chunk]))
    tasks.sort(key=lambda t: -len(members[t[0]]))  # long tasks first
    t0 = time.perf_counter()
    with _pool(workers) as pool:
        res = list(pool.map(_sample_rows, *zip(*tasks)))
    wall = time.perf_counter() - t0
    rows_s = np.zeros(len(members))
    secs = np.zeros(len(members))
    for k, r, s in res:
        rows_s[k] += r
        secs[k] += s
    return {"rows": rows_s, "seconds": secs, "wall": wall}


def schedule_makespan(el_seconds, workers: int) -> float:
    """Wall time of the reference pool on per-element single-worker times:
    FIFO in element order onto the first free worker (clustering.py:281-315)."""
    free = [0.0] * max(workers, 1)
    for t in el_seconds:
        i = int(np.argmin(free))
        free[i] += float(t)
    return max(free)
