"""Per-element DBSCAN on the GPU (mirrors nervemap/clustering.py's API).

The reference chooses, per cover element, between a precomputed cdist matrix
and on-the-fly numpy rows (clustering.py:201-208). Both evaluate the same
Euclidean distance but in different fp64 summation orders, which can flip an
eps decision at exact ties. The GPU engine never builds
either matrix; it evaluates every eps decision in the order the reference
would have used for that element (BM_ORDER_SEQUENTIAL for matrix elements,
BM_ORDER_PAIRWISE otherwise), so outputs are bit-identical for both modes,
any threshold and any budget.

`threads` is accepted for signature compatibility and validated, but never
forks (CUDA cannot survive fork); the GPU count is a separate knob
(paper_2011_03209_b200.distributed).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import DataError, MatrixBudgetExceeded

DEFAULT_PRECOMPUTE_THRESHOLD = 20_000
DEFAULT_MEM_BUDGET_BYTES = 8 << 30
MEM_BUDGET_ENV = "MAPPER_MEM_BUDGET_BYTES"
STRATEGY_MODES = ("precomputed", "on-the-fly")

# Cover elements are clustered in groups of at most this many membership
# entries per device call so cancel_check is polled between groups
# (clustering.py:273-274, 296-297). With a cancel_check, a group also holds at
# most CANCEL_GROUP_PAIRS of pair work (sum n_k^2, ~0.1 s of device time at
# cfg3's density), so a second-long build (cfg5) is polled several times;
# without one, the whole build is one call.
CANCEL_GROUP_ENTRIES = 4_000_000
CANCEL_GROUP_PAIRS = 2.0e10


def effective_mem_budget() -> int:
    raw = os.environ.get(MEM_BUDGET_ENV)
    if raw is None:
        return DEFAULT_MEM_BUDGET_BYTES
    try:
        v = int(raw)
    except ValueError:
        raise DataError(f"{MEM_BUDGET_ENV} must be an integer, got {raw!r}") from None
    if v <= 0:
        raise DataError(f"{MEM_BUDGET_ENV} must be positive")
    return v


@dataclass(frozen=True)
class DbscanParams:
    eps: float
    min_pts: int

    def __post_init__(self):
        if not self.eps > 0:
            raise DataError("eps must be positive")
        if self.min_pts < 1:
            raise DataError("min-pts must be >= 1")


@dataclass(frozen=True)
class DistanceStrategy:
    mode: str = "precomputed"
    threshold: int = DEFAULT_PRECOMPUTE_THRESHOLD

    def __post_init__(self):
        if self.mode not in STRATEGY_MODES:
            raise DataError(f"unknown strategy mode {self.mode!r}")
        if self.threshold < 1:
            raise DataError("precompute threshold must be >= 1")


@dataclass
class PullbackClustering:
    element_index: int
    clusters: list  # sorted global rows, ordered by smallest row
    noise: list

    # cluster_all's results keep their rows as flat arrays (`_lazy`: rows in
    # cluster order, cluster sizes, noise rows) until a caller first reads
    # `clusters` or `noise`; the lists are built then, once. build_graph reads
    # the flat arrays (flat_clusters), so membership -> cluster_all ->
    # build_graph never converts the ~N row ids to Python ints.
    def __getattr__(self, name):
        if name in ("clusters", "noise"):
            lazy = self.__dict__.get("_lazy")
            if lazy is not None:
                flat, sizes, noise = lazy
                cuts = np.zeros(len(sizes) + 1, dtype=np.int64)
                np.cumsum(sizes, out=cuts[1:])
                clusters = [flat[cuts[c]:cuts[c + 1]].tolist() for c in range(len(sizes))]
                self.__dict__.update(
                    clusters=clusters, noise=noise.tolist(),
                    _flat=(flat, sizes, id(clusters), [(id(c), len(c)) for c in clusters]))
                self.__dict__.pop("_lazy", None)
                return self.__dict__[name]
        raise AttributeError(f"{type(self).__name__!r} object has no attribute {name!r}")

    @classmethod
    def _from_flat(cls, element_index: int, flat: np.ndarray, sizes: np.ndarray,
                   noise: np.ndarray) -> "PullbackClustering":
        obj = cls.__new__(cls)
        obj.__dict__.update(element_index=element_index, _lazy=(flat, sizes, noise))
        return obj


@dataclass
class ClusterRunStats:
    """Telemetry (clustering.py:86-93). On the GPU path peak_matrix_bytes is
    the largest distance matrix the reference would have materialised
    (matrix-ordered elements only), so the field keeps its meaning for
    callers comparing budgets; `adjacency_bytes` is what the device used."""

    peak_matrix_bytes: int = 0
    matrix_elements: int = 0
    fallback_elements: int = 0
    per_element_rows: list = field(default_factory=list)
    pairs_evaluated: int = 0
    pairs_rechecked: int = 0
    adjacency_bytes: int = 0


def element_uses_matrix(n_rows: int, strategy: DistanceStrategy, budget: int) -> bool:
    """clustering.py:201-208 — a pure function of size, threshold, budget."""
    if strategy.mode != "precomputed":
        return False
    if n_rows > strategy.threshold:
        return False
    return n_rows * n_rows * 8 <= budget


def element_orders(sizes, strategy: DistanceStrategy, budget: int) -> np.ndarray:
    return np.array([
        _native.ORDER_SEQUENTIAL if element_uses_matrix(int(n), strategy, budget)
        else _native.ORDER_PAIRWISE for n in sizes], dtype=np.uint8)


def fill_stats(stats_out: ClusterRunStats | None, sizes, orders, strategy, dev_stats=None):
    if stats_out is None:
        return
    sizes = [int(s) for s in sizes]
    uses = [o == _native.ORDER_SEQUENTIAL for o in orders]
    stats_out.matrix_elements = sum(uses)
    stats_out.fallback_elements = sum(
        1 for k, s in enumerate(sizes) if strategy.mode == "precomputed" and s and not uses[k])
    stats_out.per_element_rows = sizes
    stats_out.peak_matrix_bytes = max(
        [s * s * 8 for k, s in enumerate(sizes) if uses[k]], default=0)
    if dev_stats is not None:
        stats_out.pairs_evaluated += int(dev_stats[0])
        stats_out.pairs_rechecked += int(dev_stats[1])
        stats_out.adjacency_bytes = max(stats_out.adjacency_bytes, int(dev_stats[4]))


def split_groups(offsets: np.ndarray, limit: int = CANCEL_GROUP_ENTRIES,
                 pair_limit: float | None = None) -> list:
    """Contiguous element ranges of bounded total size (cancel_check cadence):
    at most `limit` entries and, if given, `pair_limit` of sum n_k^2."""
    groups, k0, acc, pairs = [], 0, 0, 0.0
    n_el = len(offsets) - 1
    for k in range(n_el):
        nk = int(offsets[k + 1] - offsets[k])
        if acc and (acc + nk > limit or
                    (pair_limit is not None and pairs + float(nk) ** 2 > pair_limit)):
            groups.append((k0, k))
            k0, acc, pairs = k, 0, 0.0
        acc += nk
        pairs += float(nk) ** 2
    groups.append((k0, n_el))
    return groups


def cluster_device(X, rows_dev, offsets, params: DbscanParams, orders, cancel_check=None,
                   engine: int = _native.ENGINE_AUTO):
    """Cluster every element of a device membership; returns (labels_dev,
    n_clusters host, device stats). Polls cancel_check between groups."""
    import torch

    from . import engine as eng

    n_el = len(offsets) - 1
    labels = torch.empty(max(int(offsets[-1]), 1), dtype=torch.int32, device=X.device)
    ncl = np.zeros(n_el, dtype=np.int32)
    stats = np.zeros(8, dtype=np.int64)
    pair_limit = CANCEL_GROUP_PAIRS if cancel_check is not None else None
    for k0, k1 in split_groups(offsets, CANCEL_GROUP_ENTRIES, pair_limit):
        if cancel_check is not None:
            cancel_check()
        a, b = int(offsets[k0]), int(offsets[k1])
        sub_off = offsets[k0:k1 + 1] - a
        if b == a:
            continue
        lab, nc, st = eng.cluster(X, rows_dev[a:b], sub_off, params.eps, params.min_pts,
                                  orders[k0:k1], engine)
        labels[a:b] = lab
        ncl[k0:k1] = nc
        stats[:4] += st[:4]
        stats[4] = max(stats[4], st[4])
        stats[5:] += st[5:]
    return labels[: int(offsets[-1])], ncl, stats


def labels_to_clusterings(rows_h: np.ndarray, offsets: np.ndarray, labels_h: np.ndarray,
                          ncl: np.ndarray) -> list:
    """Per-element PullbackClustering lists from per-entry cluster ranks."""
    out = []
    for k in range(len(offsets) - 1):
        r = rows_h[offsets[k]:offsets[k + 1]]
        lab = labels_h[offsets[k]:offsets[k + 1]]
        if ncl[k]:
            order = np.argsort(lab, kind="stable")
            lab_sorted = lab[order]
            rows_sorted = r[order]
            cuts = np.searchsorted(lab_sorted, np.arange(int(ncl[k]) + 1))
            clusters = [rows_sorted[cuts[c]:cuts[c + 1]].tolist() for c in range(int(ncl[k]))]
        else:
            rows_sorted, cuts = r[:0], np.zeros(1, dtype=np.int64)
            clusters = []
        noise = r[lab < 0].tolist()
        pbc = PullbackClustering(k, clusters, noise)
        # flat copy for build_graph's fast path (no list -> array conversion);
        # only used while pbc.clusters still holds these very lists
        pbc._flat = (rows_sorted[cuts[0]:cuts[-1]], np.diff(cuts), id(clusters),
                     [(id(c), len(c)) for c in clusters])
        out.append(pbc)
    return out


def grouped_clusterings(rows_h: np.ndarray, offsets: np.ndarray, labels_h: np.ndarray,
                        ncl: np.ndarray, node_rows_h: np.ndarray, node_off_h: np.ndarray) -> list:
    """Per-element PullbackClustering lists from the device's node grouping
    (bm_group_nodes: rows of every cluster, ascending, in (element, cluster)
    order) — the host only slices (the Python lists are built on first
    access); noise rows come from one mask pass."""
    n_el = len(offsets) - 1
    noise_idx = np.flatnonzero(labels_h < 0)
    nb = np.searchsorted(noise_idx, offsets)
    node0 = np.zeros(n_el + 1, dtype=np.int64)
    np.cumsum(np.asarray(ncl, dtype=np.int64), out=node0[1:])
    out = []
    for k in range(n_el):
        v0, v1 = int(node0[k]), int(node0[k + 1])
        a, b = int(node_off_h[v0]), int(node_off_h[v1])
        out.append(PullbackClustering._from_flat(k, node_rows_h[a:b],
                                                 np.diff(node_off_h[v0:v1 + 1]),
                                                 rows_h[noise_idx[nb[k]:nb[k + 1]]]))
    return out


def flat_clusters(pbc):
    """(rows in cluster order, cluster sizes) of a PullbackClustering made by
    cluster_all, or None if its cluster lists were replaced or resized."""
    lazy = pbc.__dict__.get("_lazy")
    if lazy is not None:  # lists never built: the flat arrays are the truth
        return lazy[0], lazy[1]
    f = pbc.__dict__.get("_flat")
    if f is None or f[2] != id(pbc.clusters) or len(pbc.clusters) != len(f[3]):
        return None
    for c, (ic, ln) in zip(pbc.clusters, f[3]):
        if id(c) != ic or len(c) != ln:
            return None
    return f[0], f[1]


def cluster_all(pc, memberships: list, params: DbscanParams, strategy: DistanceStrategy,
                threads: int = 1, budget_bytes: int | None = None,
                stats_out: ClusterRunStats | None = None, cancel_check=None,
                engine: int = _native.ENGINE_AUTO) -> list:
    """One PullbackClustering per cover element (clustering.py:238-316), on the GPU."""
    import torch

    from .device import cached_device_array, require_gpu

    if threads < 1:
        raise DataError("threads must be >= 1")
    budget = effective_mem_budget() if budget_bytes is None else budget_bytes
    sizes = [int(np.asarray(r).size) for r in memberships]
    orders = element_orders(sizes, strategy, budget)
    n_el = len(memberships)
    if n_el == 0:
        fill_stats(stats_out, sizes, orders, strategy)
        return []
    offsets = np.zeros(n_el + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    rows_h = (np.concatenate([np.asarray(r, dtype=np.int64) for r in memberships])
              if offsets[-1] else np.zeros(0, dtype=np.int64))
    if offsets[-1] == 0:
        fill_stats(stats_out, sizes, orders, strategy)
        if cancel_check is not None:
            cancel_check()
        return [PullbackClustering(k, [], []) for k in range(n_el)]
    if rows_h.min() < 0 or rows_h.max() >= pc.n_rows:
        raise DataError("membership row out of range")
    dev = require_gpu()
    X = cached_device_array(pc, pc.points, dev)
    rows_dev = torch.from_numpy(rows_h).to(dev)
    labels, ncl, st = cluster_device(X, rows_dev, offsets, params, orders, cancel_check, engine)
    fill_stats(stats_out, sizes, orders, strategy, st)
    from . import engine as eng

    node_rows, node_off, _ = eng.group_nodes(rows_dev, offsets, labels, ncl)
    return grouped_clusterings(rows_h, offsets, labels.cpu().numpy(), ncl,
                               node_rows.cpu().numpy(), node_off.cpu().numpy())


def dbscan_rows(pc, rows, params: DbscanParams, order: int = _native.ORDER_SEQUENTIAL,
                element_index: int = 0, engine: int = _native.ENGINE_AUTO) -> PullbackClustering:
    """DBSCAN over one pullback set (clustering.py:151-198) in the given exact order."""
    import torch

    from .device import cached_device_array, require_gpu

    rows_h = np.asarray(rows, dtype=np.int64)
    if rows_h.size == 0:
        return PullbackClustering(element_index, [], [])
    dev = require_gpu()
    X = cached_device_array(pc, pc.points, dev)
    offsets = np.array([0, rows_h.size], dtype=np.int64)
    labels, ncl, _ = cluster_device(X, torch.from_numpy(rows_h).to(dev), offsets, params,
                                    np.array([order], dtype=np.uint8), None, engine)
    out = labels_to_clusterings(rows_h, offsets, labels.cpu().numpy(), ncl)[0]
    out.element_index = element_index
    return out


def pairwise_distances(pc, rows, budget_bytes: int | None = None,
                       order: int = _native.ORDER_SEQUENTIAL) -> np.ndarray:
    """Full distance matrix over `rows` (clustering.py:96-113), computed on the
    GPU in the exact cdist order (or numpy's pairwise order). Budget semantics
    are the reference's: MatrixBudgetExceeded when rows^2*8 > budget. Not on the
    hot path: the DBSCAN engine never materialises distance matrices."""
    import torch

    from .device import cached_device_array, require_gpu, stream_ptr

    rows = np.asarray(rows)
    if rows.size == 0:
        raise DataError("rows must be nonempty")
    budget = effective_mem_budget() if budget_bytes is None else budget_bytes
    need = int(rows.size) * int(rows.size) * 8
    if need > budget:
        raise MatrixBudgetExceeded(
            f"{rows.size}^2 distance matrix needs {need} bytes, budget {budget}")
    dev = require_gpu()
    X = cached_device_array(pc, pc.points, dev)
    r = torch.from_numpy(rows.astype(np.int64)).to(dev)
    out = torch.empty((rows.size, rows.size), dtype=torch.float64, device=dev)
    rc = _native.load().bm_pairwise_distances(_native.ptr(X), X.shape[0], X.shape[1],
                                              _native.ptr(r), rows.size, order,
                                              _native.ptr(out), stream_ptr(dev))
    _native.check(rc, "pairwise distances")
    return out.cpu().numpy()
