"""ORACLE (TEST INFRASTRUCTURE ONLY) — chunked DBSCAN for elements too large
for a dense n_k x n_k matrix.

Same semantics as mapper_oracle.dbscan_element (restating
/root/reference/pkg/src/nervemap/clustering.py:151-198: core = count >= min_pts
including self; clusters = components of core points under the eps relation;
a non-core point takes the cluster of its smallest-index core neighbour;
clusters ordered by smallest member), but the distances are evaluated in row
blocks of the upper triangle and only the eps-pairs are kept, so the memory
is O(block * n + eps-edges) instead of O(n^2).

Distances use the reference's own arithmetic:
  ORDER_SEQUENTIAL  scipy cdist (clustering.py:113) on (block, rows >= block)
  ORDER_PAIRWISE    numpy sqrt(((P - P[i])**2).sum(axis=-1)) (clustering.py:137-139)
A pair (i, j) and (j, i) get bitwise equal distances in both orders
((a-b)^2 == (b-a)^2 exactly in IEEE fp64), so the upper triangle suffices.

Pinned in tests/test_oracle.py against the dense oracle and the reference's
golden graphs. Only tests/, smoke() and bench.py's CPU legs use this module.
"""

from __future__ import annotations

import multiprocessing as mp
from concurrent.futures import ProcessPoolExecutor

import numpy as np
from scipy.sparse import coo_matrix
from scipy.sparse.csgraph import connected_components
from scipy.spatial.distance import cdist

ORDER_SEQUENTIAL = 0
ORDER_PAIRWISE = 1

_CTX: dict = {}


def _init(ctx):
    _CTX.clear()
    _CTX.update(ctx)


def _block_pairs(i0: int, i1: int):
    """eps-pairs (i, j), i0 <= i < i1, j > i, of the current element."""
    P, eps, order = _CTX["P"], _CTX["eps"], _CTX["order"]
    if order == ORDER_SEQUENTIAL:
        D = cdist(P[i0:i1], P[i0:])
    else:
        D = np.empty((i1 - i0, P.shape[0] - i0))
        T = P[i0:]
        for a in range(i0, i1):
            diff = T - P[a]
            D[a - i0] = np.sqrt((diff * diff).sum(axis=1))
    m = D <= eps
    del D
    # strict upper triangle: column c (global i0 + c) > row i0 + a  <=> c > a
    m &= np.arange(m.shape[1])[None, :] > np.arange(m.shape[0])[:, None]
    a, c = np.nonzero(m)
    return (a + i0).astype(np.int32), (c + i0).astype(np.int32)


def eps_pairs(P: np.ndarray, eps: float, order: int, block: int = 1024,
              workers: int = 1) -> tuple:
    """All eps-pairs i < j of the rows of P (int32 arrays, ascending i)."""
    n = P.shape[0]
    if order == ORDER_PAIRWISE:
        block = min(block, 64)
    blocks = [(i0, min(n, i0 + block)) for i0 in range(0, n, block)]
    ctx = {"P": P, "eps": eps, "order": order}
    if workers <= 1 or len(blocks) <= 1:
        _init(ctx)
        res = [_block_pairs(*b) for b in blocks]
    else:
        with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork"),
                                 initializer=_init, initargs=(ctx,)) as pool:
            res = list(pool.map(_block_pairs, *zip(*blocks)))
    if not res:
        return np.zeros(0, np.int32), np.zeros(0, np.int32)
    return (np.concatenate([r[0] for r in res]), np.concatenate([r[1] for r in res]))


def labels_from_pairs(n: int, I: np.ndarray, J: np.ndarray, min_pts: int) -> np.ndarray:
    """Cluster rank per point (ordered by smallest member) or -1, from the
    eps-pairs i < j (clustering.py:151-198 semantics, as union-find)."""
    counts = np.ones(n, dtype=np.int64)  # self (d = 0 <= eps)
    np.add.at(counts, I, 1)
    np.add.at(counts, J, 1)
    core = counts >= min_pts
    root = np.full(n, -1, dtype=np.int64)
    ci = np.flatnonzero(core)
    if ci.size == 0:
        return root
    both = core[I] & core[J]
    g = coo_matrix((np.ones(int(both.sum()), dtype=np.int8), (I[both], J[both])),
                   shape=(n, n)).tocsr()
    _, comp = connected_components(g, directed=False)
    first = np.full(comp.max() + 1, n, dtype=np.int64)
    np.minimum.at(first, comp[ci], ci)
    root[ci] = first[comp[ci]]
    # border: smallest-index core neighbour
    bmin = np.full(n, n, dtype=np.int64)
    s = core[J] & ~core[I]
    np.minimum.at(bmin, I[s], J[s])
    s = core[I] & ~core[J]
    np.minimum.at(bmin, J[s], I[s])
    bord = np.flatnonzero(~core & (bmin < n))
    root[bord] = root[bmin[bord]]
    lab = np.full(n, -1, dtype=np.int64)
    idx = np.flatnonzero(root >= 0)
    # cluster ids by smallest member: the first index carrying each root
    uroots, first_idx = np.unique(root[idx], return_index=True)
    rank_of = np.empty(len(uroots), dtype=np.int64)
    rank_of[np.argsort(idx[first_idx], kind="stable")] = np.arange(len(uroots))
    lab[idx] = rank_of[np.searchsorted(uroots, root[idx])]
    return lab


def dbscan_element(X: np.ndarray, rows: np.ndarray, eps: float, min_pts: int, order: int,
                   block: int = 1024, workers: int = 1) -> tuple:
    """(clusters as lists of global rows, noise list) — chunked, exact."""
    rows = np.asarray(rows, dtype=np.int64)
    if rows.size == 0:
        return [], []
    P = np.ascontiguousarray(X[rows])
    I, J = eps_pairs(P, eps, order, block, workers)
    lab = labels_from_pairs(rows.size, I, J, min_pts)
    ncl = int(lab.max()) + 1 if lab.size else 0
    if ncl:
        o = np.argsort(lab, kind="stable")
        ls = lab[o]
        cuts = np.searchsorted(ls, np.arange(ncl + 1))
        clusters = [rows[o[cuts[c]:cuts[c + 1]]].tolist() for c in range(ncl)]
    else:
        clusters = []
    return clusters, rows[lab < 0].tolist()
