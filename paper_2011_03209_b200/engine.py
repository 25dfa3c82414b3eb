"""Device-resident stage functions over torch tensors (thin layer on the C ABI).

Each function launches on the current torch stream of the tensors' device
and returns device tensors; host arrays come back only where the reference
API needs them (per-element counts, cluster counts, edges). The public API
modules (filters, cover, clustering, nerve, pipeline) are built from these.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .device import stream_ptr
from .errors import DataError

P = _native.ptr


def lens(X: torch.Tensor, kind: int, col: int = 0) -> torch.Tensor:
    """K1 (filters.py:133-140): one lens column of N fp64 values."""
    n, d = X.shape
    out = torch.empty(n, dtype=torch.float64, device=X.device)
    rc = _native.load().bm_lens_f64(kind, P(X), n, d, col, P(out), stream_ptr(X.device))
    _native.check(rc, "lens")
    return out


def pairwise_lens(X: torch.Tensor, kind: int, param: float, qrows=None, trows=None) -> torch.Tensor:
    """O(N x M) lens values (filters.py:103-150) of the query rows (default:
    all) against the target rows (default: all); see bm_pairwise_lens."""
    n, d = X.shape
    nq = n if qrows is None else int(qrows.numel())
    m = n if trows is None else int(trows.numel())
    out = torch.empty(max(nq, 1), dtype=torch.float64, device=X.device)
    rc = _native.load().bm_pairwise_lens(int(kind), ctypes.c_double(float(param)), P(X), n, d,
                                         P(qrows), nq, P(trows), m, P(out),
                                         stream_ptr(X.device))
    _native.check(rc, "pairwise lens")
    return out[:nq]


def mean_1d(v: torch.Tensor) -> torch.Tensor:
    """numpy's 1-D mean (pairwise sum / n) of a device vector, as a 1-element
    device tensor (bm_node_stats' filter-mean path with one node)."""
    n = int(v.numel())
    rows = torch.arange(n, dtype=torch.int64, device=v.device)
    off = torch.tensor([0, n], dtype=torch.int64, device=v.device)
    fm = torch.empty(1, dtype=torch.float64, device=v.device)
    rc = _native.load().bm_node_stats(0, 1, P(v.contiguous()), 1, P(rows), P(off), 1, 0, P(fm),
                                      stream_ptr(v.device))
    _native.check(rc, "mean")
    return fm


def normalize(X: torch.Tensor, scheme: str) -> torch.Tensor:
    """dataset.py:165-186 on the device; 'none' returns X itself."""
    if scheme == "none":
        return X
    code = {"minmax": 1, "l2": 2}.get(scheme)
    if code is None:
        raise DataError(f"unknown normalization {scheme!r}")
    n, d = X.shape
    out = torch.empty_like(X)
    rc = _native.load().bm_normalize_f64(code, P(X), n, d, P(out), stream_ptr(X.device))
    _native.check(rc, "normalize")
    return out


def cover_tables(cover) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    lo = np.array([iv.lo for axis in cover.axes for iv in axis], dtype=np.float64)
    hi = np.array([iv.hi for axis in cover.axes for iv in axis], dtype=np.float64)
    n_axis = np.array([len(axis) for axis in cover.axes], dtype=np.int32)
    return lo, hi, n_axis


def membership(F: torch.Tensor, cover) -> tuple[torch.Tensor, np.ndarray]:
    """K2 (cover.py:122-140): rows of every element, ascending, concatenated.

    F is the (N, m) fp64 lens matrix on the device. Returns (rows_dev int64,
    offsets_host int64[n_el+1]).
    """
    F = F.contiguous()
    n, m = F.shape
    lo, hi, n_axis = cover_tables(cover)
    n_el = int(np.prod(n_axis))
    counts = np.zeros(n_el, dtype=np.int64)
    lib = _native.load()
    s = stream_ptr(F.device)
    rc = lib.bm_membership_count(P(F), n, m, P(lo), P(hi), P(n_axis), P(counts), s)
    _native.check(rc, "membership count")
    offsets = np.zeros(n_el + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    rows = torch.empty(int(offsets[-1]), dtype=torch.int64, device=F.device)
    d_off = torch.from_numpy(offsets).to(F.device)
    rc = lib.bm_membership_fill(P(F), n, m, P(lo), P(hi), P(n_axis), P(d_off), P(rows), s)
    _native.check(rc, "membership fill")
    return rows, offsets


def cluster(X: torch.Tensor, rows: torch.Tensor, offsets: np.ndarray, eps: float, min_pts: int,
            orders: np.ndarray, engine: int = _native.ENGINE_AUTO):
    """K3..K6 (clustering.py:151-198) for every element at once.

    Returns (labels_dev int32 per membership entry: cluster rank inside its
    element or -1, n_clusters host int32[n_el], stats host int64[8]).
    """
    n, d = X.shape
    n_el = len(offsets) - 1
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    orders = np.ascontiguousarray(orders, dtype=np.uint8)
    labels = torch.empty(max(int(offsets[-1]), 1), dtype=torch.int32, device=X.device)
    ncl = np.zeros(max(n_el, 1), dtype=np.int32)
    stats = np.zeros(8, dtype=np.int64)
    rc = _native.load().bm_cluster_elements(
        P(X), n, d, P(rows), P(offsets), n_el, ctypes.c_double(float(eps)), int(min_pts),
        P(orders), int(engine), P(labels), P(ncl), P(stats), stream_ptr(X.device))
    _native.check(rc, "cluster elements")
    return labels[: int(offsets[-1])], ncl[:n_el], stats


def element_work(X: torch.Tensor, rows: torch.Tensor, offsets: np.ndarray, eps: float):
    """Kept (unpruned) tile pairs per element: the distance work the engine
    will do (bm_element_work); host int64[n_el]."""
    n, d = X.shape
    n_el = len(offsets) - 1
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    out = np.zeros(max(n_el, 1), dtype=np.int64)
    rc = _native.load().bm_element_work(P(X), n, d, P(rows), P(offsets), n_el,
                                        ctypes.c_double(float(eps)), P(out), stream_ptr(X.device))
    _native.check(rc, "element work")
    return out[:n_el]


class BigElement:
    """Row-block protocol handle for ONE cover element sharded over ranks
    (include/b200map.h bm_big_*). Arrays cnt/par/bmin hold
    `padded` int32 entries; every call runs on the stream current at open."""

    TILE = 128

    def __init__(self, X: torch.Tensor, rows: torch.Tensor, eps: float, min_pts: int, order: int,
                 engine: int = _native.ENGINE_AUTO):
        n, d = X.shape
        self._lib = _native.load()
        self._h = ctypes.c_void_p()
        tiles = ctypes.c_int64(0)
        self.device = X.device
        self.n_rows = int(rows.numel())
        rc = self._lib.bm_big_open(P(X), n, d, P(rows), self.n_rows, ctypes.c_double(float(eps)),
                                   int(min_pts), int(order), int(engine), stream_ptr(X.device),
                                   ctypes.byref(self._h), ctypes.byref(tiles))
        _native.check(rc, "big element open")
        self.tiles = int(tiles.value)
        self.padded = self.tiles * self.TILE

    def zeros(self) -> torch.Tensor:
        return torch.zeros(self.padded, dtype=torch.int32, device=self.device)

    def counts(self, I0: int, I1: int, cnt: torch.Tensor) -> None:
        _native.check(self._lib.bm_big_counts(self._h, int(I0), int(I1), P(cnt)), "big counts")

    def init(self, cnt: torch.Tensor, par: torch.Tensor, bmin: torch.Tensor) -> None:
        _native.check(self._lib.bm_big_init(self._h, P(cnt), P(par), P(bmin)), "big init")

    def components(self, I0: int, I1: int, par: torch.Tensor, bmin: torch.Tensor) -> None:
        _native.check(self._lib.bm_big_components(self._h, int(I0), int(I1), P(par), P(bmin)),
                      "big components")

    def labels(self, par: torch.Tensor, bmin: torch.Tensor):
        out = torch.empty(max(self.n_rows, 1), dtype=torch.int32, device=self.device)
        ncl = np.zeros(1, dtype=np.int32)
        _native.check(self._lib.bm_big_labels(self._h, P(par), P(bmin), P(out), P(ncl)),
                      "big labels")
        return out[: self.n_rows], int(ncl[0])

    def row_tiles(self) -> np.ndarray:
        """Kept tile pairs before each tile row (tiles + 1 entries)."""
        out = np.zeros(self.tiles + 1, dtype=np.int64)
        _native.check(self._lib.bm_big_row_tiles(self._h, P(out)), "big row tiles")
        return out

    def stats(self) -> np.ndarray:
        st = np.zeros(8, dtype=np.int64)
        _native.check(self._lib.bm_big_stats(self._h, P(st)), "big stats")
        return st

    def close(self) -> None:
        if self._h:
            _native.check(self._lib.bm_big_close(self._h), "big close")
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def merge_forest(par: torch.Tensor, other: torch.Tensor) -> None:
    """par := union of the union-find forests par and other (same length)."""
    rc = _native.load().bm_merge_forest(P(par), P(other), int(par.numel()),
                                        stream_ptr(par.device))
    _native.check(rc, "merge forest")


def group_nodes(rows: torch.Tensor, offsets: np.ndarray, labels: torch.Tensor,
                n_clusters: np.ndarray):
    """Node row lists in (element, cluster) order (nerve.py:84-101)."""
    n_el = len(offsets) - 1
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    ncl = np.ascontiguousarray(n_clusters, dtype=np.int32)
    n_nodes = int(ncl.sum())
    dev = rows.device
    node_rows = torch.empty(max(int(offsets[-1]), 1), dtype=torch.int64, device=dev)
    node_off = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
    total = ctypes.c_int64(0)
    rc = _native.load().bm_group_nodes(P(rows), P(offsets), n_el, P(labels), P(ncl),
                                       P(node_rows), P(node_off), ctypes.byref(total),
                                       stream_ptr(dev))
    _native.check(rc, "group nodes")
    return node_rows[: total.value], node_off, n_nodes


def nerve_edges(node_rows: torch.Tensor, node_off: torch.Tensor, n_nodes: int,
                n_points: int) -> np.ndarray:
    """K7 (nerve.py:103-113): sorted (s, t, w) int64 array of shape (E, 3)."""
    lib = _native.load()
    s = stream_ptr(node_off.device)
    ne = ctypes.c_int64(0)
    max_edges = n_nodes * (n_nodes - 1) // 2
    if 0 < max_edges <= (1 << 22):
        # a buffer for every possible edge: one call computes and writes them
        edges = torch.empty((max_edges, 3), dtype=torch.int64, device=node_off.device)
        rc = lib.bm_nerve_edges(P(node_rows), P(node_off), n_nodes, n_points, P(edges),
                                ctypes.byref(ne), s)
        _native.check(rc, "nerve edges")
        return edges[: ne.value].cpu().numpy()
    rc = lib.bm_nerve_edges(P(node_rows), P(node_off), n_nodes, n_points, None,
                            ctypes.byref(ne), s)
    _native.check(rc, "nerve edges (count)")
    if ne.value == 0:
        return np.zeros((0, 3), dtype=np.int64)
    edges = torch.empty((ne.value, 3), dtype=torch.int64, device=node_off.device)
    rc = lib.bm_nerve_edges(P(node_rows), P(node_off), n_nodes, n_points, P(edges),
                            ctypes.byref(ne), s)
    _native.check(rc, "nerve edges")
    return edges.cpu().numpy()


def node_payload(X: torch.Tensor, F: torch.Tensor, node_rows: torch.Tensor,
                 node_off: torch.Tensor, n_nodes: int):
    """Per-node column means and filter means (nerve.py:60-62, 96)."""
    d = X.shape[1]
    m = F.shape[1]
    dev = X.device
    stats = torch.empty((max(n_nodes, 1), d), dtype=torch.float64, device=dev)
    fmean = torch.empty((max(n_nodes, 1), m), dtype=torch.float64, device=dev)
    lib = _native.load()
    s = stream_ptr(dev)
    for v0 in range(0, n_nodes, 65535):
        cnt = min(65535, n_nodes - v0)
        rc = lib.bm_node_stats(P(X), d, P(F.contiguous()), m, P(node_rows),
                               P(node_off) + 8 * v0, cnt, P(stats) + 8 * d * v0,
                               P(fmean) + 8 * m * v0, s)
        _native.check(rc, "node stats")
    return stats[:n_nodes], fmean[:n_nodes]
