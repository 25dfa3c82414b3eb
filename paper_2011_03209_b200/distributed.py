"""Multi-GPU Mapper build: cover elements sharded across ranks (one process
per GPU, torch.distributed over NCCL), cluster memberships gathered to rank 0.

This replaces the reference's only parallelism strategy, the fork pool over
cover elements (clustering.py:281-315): elements are independent DBSCAN
instances, so the work partitions with no data-path collective; the single
exchange is the gather of per-entry cluster labels to the rank that builds
nodes and edges.

An element too large for LPT to balance (n_k^2 above 1/world of the total)
or for one device's memory is instead split by ROW BLOCKS of its triangular
eps-graph: ranks take tile-row windows of equal tile
area, all-reduce(sum) the eps-neighbour counts, union their windows'
core-core bits locally, and rank 0 merges the forests and the all-reduced
(min) border choices into the labels (`rowblock_cluster`).

Every rank holds X and evaluates the (cheap, HBM-bound) lens and cover
itself, so memberships are identical on all ranks without communication.
Elements are assigned by LPT on the pair work n_k^2 (largest first onto the
least-loaded rank), a pure function of the sizes, so the assignment — and the
output — does not depend on the number of ranks or on timing.
"""

from __future__ import annotations

import heapq

import numpy as np


def lpt_partition(sizes, world: int, costs=None) -> list:
    """Element ids per rank, largest cost first onto the least-loaded rank
    (cost: `costs` if given, else n_k^2); empty elements are skipped."""
    cost = [float(c) for c in costs] if costs is not None else [float(s) ** 2 for s in sizes]
    loads = [(0.0, r) for r in range(world)]
    heapq.heapify(loads)
    parts = [[] for _ in range(world)]
    order = sorted(range(len(sizes)), key=lambda k: (-cost[k], k))
    for k in order:
        if int(sizes[k]) == 0:
            continue
        load, r = heapq.heappop(loads)
        parts[r].append(k)
        heapq.heappush(loads, (load + cost[k], r))
    return [sorted(p) for p in parts]


# Cost model for scheduling (measured at cfg3 on one B200): a kept 128 x 128
# tile pair costs ~16 ns of distance work; the per-row stages (grouping,
# quantisation, components, relabel) ~0.7 us per 128-row tile, i.e. ~45 kept
# tile pairs' worth.
ROW_TILE_COST = 45


def element_costs(X, rows, offsets, sizes, eps, rank: int, world: int, dist) -> np.ndarray:
    """Per-element scheduling cost: kept (unpruned) tile pairs, from the
    engine's own pruning (bm_element_work), plus ROW_TILE_COST per row tile.
    Each rank estimates a 1/world share of the elements (round-robin by size)
    and one all_reduce(sum) gives every rank every estimate."""
    import torch

    from . import engine as eng

    n_el = len(sizes)
    order = sorted(range(n_el), key=lambda k: (-int(sizes[k]), k))
    mine = sorted(k for i, k in enumerate(order) if i % world == rank and sizes[k] > 0)
    est = torch.zeros(max(n_el, 1), dtype=torch.int64, device=X.device)
    if mine:
        ranges, loc = pack_local(offsets, mine)
        rows_loc = torch.cat([rows[a:b] for a, b in ranges])
        kept = eng.element_work(X, rows_loc, loc, eps)
        est[torch.as_tensor(mine, device=X.device)] = torch.from_numpy(kept).to(X.device)
    if world > 1:
        dist.all_reduce(est, op=dist.ReduceOp.SUM)
    kept = est.cpu().numpy()[:n_el]
    tiles = -(-np.asarray(sizes, dtype=np.int64) // 128)
    return kept + ROW_TILE_COST * tiles


def pack_local(offsets: np.ndarray, elems: list) -> tuple:
    """(entry ranges, local offsets) of a rank's elements, in element order."""
    ranges = [(int(offsets[k]), int(offsets[k + 1])) for k in elems]
    loc = np.zeros(len(elems) + 1, dtype=np.int64)
    np.cumsum([b - a for a, b in ranges], out=loc[1:])
    return ranges, loc


def gather_labels(labels_local, ncl_local, elems: list, parts: list, offsets: np.ndarray,
                  n_el: int, rank: int, world: int, dist, device):
    """All ranks contribute their elements' labels; rank 0 returns the full
    per-entry label array and per-element cluster counts (others: None).

    Collective: one gather to rank 0 of a fixed-size int32 buffer per rank
    (labels padded to the largest rank, cluster counts appended); only rank 0
    builds nodes and edges, so no other rank receives anything."""
    import torch

    sizes = [int(sum(int(offsets[k + 1] - offsets[k]) for k in p)) for p in parts]
    cap = max(max(sizes), 1) + max(len(p) for p in parts)
    buf = torch.full((cap,), -1, dtype=torch.int32, device=device)
    n_loc = sizes[rank]
    if n_loc:
        buf[:n_loc] = labels_local[:n_loc]
    if elems:
        buf[n_loc:n_loc + len(elems)] = torch.as_tensor(np.asarray(ncl_local, dtype=np.int32),
                                                       device=device)
    out = _gather_to_root(buf, rank, world, dist)
    if rank != 0:
        return None, None
    total = int(offsets[-1])
    full = torch.empty(max(total, 1), dtype=torch.int32, device=device)
    ncl = np.zeros(n_el, dtype=np.int32)
    host_out = None
    for r in range(world):
        pos = 0
        for k in parts[r]:
            a, b = int(offsets[k]), int(offsets[k + 1])
            full[a:b] = out[r, pos:pos + (b - a)]
            pos += b - a
        if parts[r]:
            if host_out is None:
                host_out = out[:, :].cpu().numpy()
            ncl[parts[r]] = host_out[r, sizes[r]:sizes[r] + len(parts[r])]
    return full[:total], ncl


def tri_rows(T: int, I: int) -> int:
    """Tile pairs (I', J >= I') in tile rows [0, I) of a T-tile triangle."""
    return I * T - I * (I - 1) // 2


def area_windows(T: int, world: int) -> list:
    """Tile-row windows [I0, I1) per rank with (nearly) equal tile area;
    empty windows (I0 == I1) when T < world."""
    total = tri_rows(T, T)
    cuts = [0]
    I = 0
    for r in range(1, world):
        target = total * r / world
        while I < T and tri_rows(T, I + 1) <= target:
            I += 1
        if I < T and tri_rows(T, I + 1) - target < target - tri_rows(T, I):
            I += 1  # nearest cut: every window is within one tile row of its share
        cuts.append(max(I, cuts[-1]))
    cuts.append(T)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def split_window(I0: int, I1: int, T: int, max_tiles: int) -> list:
    """Sub-windows of [I0, I1) holding at most max_tiles tile pairs (>= 1 row each)."""
    out = []
    I = I0
    while I < I1:
        J, acc = I, 0
        while J < I1 and (J == I or acc + (T - J) <= max_tiles):
            acc += T - J
            J += 1
        out.append((I, J))
        I = J
    return out


def big_elements(sizes, world: int, costs=None) -> list:
    """Elements whose work (costs, else n_k^2) exceeds 1/world of the total:
    row-blocked."""
    if world <= 1:
        return []
    work = [float(c) for c in costs] if costs is not None else [float(s) ** 2 for s in sizes]
    total = sum(work)
    return [k for k, w in enumerate(work) if total > 0 and w > total / world]


def kept_windows(row_first, world: int) -> list:
    """Tile-row windows [I0, I1) per rank with (nearly) equal KEPT tile pairs;
    row_first[I] = kept pairs before tile row I (T + 1 entries)."""
    rf = np.asarray(row_first, dtype=np.float64)
    T = len(rf) - 1
    total = rf[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        I = int(np.searchsorted(rf, target))  # first I with rf[I] >= target
        if I > 0 and target - rf[I - 1] < rf[min(I, T)] - target:
            I -= 1
        cuts.append(min(max(I, cuts[-1]), T))
    cuts.append(T)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def split_window_kept(I0: int, I1: int, row_first, max_tiles: int) -> list:
    """Sub-windows of [I0, I1) holding at most max_tiles kept tile pairs
    (>= 1 row each)."""
    out = []
    I = I0
    while I < I1:
        J = I + 1
        while J < I1 and row_first[J + 1] - row_first[I] <= max_tiles:
            J += 1
        out.append((I, J))
        I = J
    return out


def _gather_to_root(t, rank: int, world: int, dist):
    """(world, *t.shape) on rank 0 (None elsewhere): one gather collective."""
    import torch

    if world == 1:
        return t.unsqueeze(0)
    out = (torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
           if rank == 0 else None)
    dist.gather(t, list(out.unbind(0)) if rank == 0 else None, dst=0)
    return out


def rowblock_cluster(be, rank: int, world: int, dist, max_tiles: int, merge_forest):
    """DBSCAN of one element split over ranks by tile-row windows.

    `be` provides the per-rank steps (engine.BigElement on a GPU; a numpy
    model in the CPU tests): counts -> all_reduce(sum) -> init -> components
    (resident window first) -> forests gathered and merged on rank 0,
    all_reduce(min) of border minima -> labels on rank 0. Returns
    (labels, n_clusters) on rank 0, (None, None) elsewhere. The result is the
    element's unique DBSCAN labelling, identical for every world size."""
    if hasattr(be, "row_tiles"):  # balanced on the kept (unpruned) tile pairs
        rf = be.row_tiles()
        I0, I1 = kept_windows(rf, world)[rank]
        wins = split_window_kept(I0, I1, rf, max_tiles) if I1 > I0 else []
    else:
        I0, I1 = area_windows(be.tiles, world)[rank]
        wins = split_window(I0, I1, be.tiles, max_tiles) if I1 > I0 else []
    cnt = be.zeros()
    for w in wins:
        be.counts(w[0], w[1], cnt)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    par, bmin = be.zeros(), be.zeros()
    be.init(cnt, par, bmin)
    for w in reversed(wins):  # the last window's bits are still resident
        be.components(w[0], w[1], par, bmin)
    dist.all_reduce(bmin, op=dist.ReduceOp.MIN)
    forests = _gather_to_root(par, rank, world, dist)
    if rank != 0:
        return None, None
    for r in range(1, world):
        merge_forest(par, forests[r])
    return be.labels(par, bmin)


def device_window_tiles(device, d: int, rows: int) -> int:
    """Largest row window (tile pairs) that fits next to the element's rows."""
    import torch

    from . import _native

    with torch.cuda.device(device):
        free = np.zeros(1, dtype=np.int64)
        _native.check(_native.load().bm_device_free_bytes(_native.ptr(free)), "free bytes")
        free = int(free[0])
    row_bytes = rows * (d * 11.0 + 64)
    return max(1, int((0.85 * free - row_bytes - (4 << 30)) / 2056))


def build_distributed(X, pc, params, rank: int, world: int, dist, budget_bytes=None,
                      engine: int = 0, cancel_check=None, balance: str = "kept", F=None):
    """Sharded hot path. Returns (DeviceGraph, stats) on rank 0 and
    (None, stats) elsewhere. balance="kept": elements and row-block windows
    are balanced on the engine's kept tile pairs (element_costs); "area": on
    n_k^2 / triangle area. cancel_check is polled by rank 0 between phases
    (a raise there aborts the other ranks at their next collective)."""
    import torch

    from . import engine as eng
    from .clustering import DbscanParams, cluster_device, effective_mem_budget, element_orders
    from .cover import build_cover_from_range
    from .filters import evaluate_device
    from .pipeline import DeviceGraph

    if F is None:  # else: the caller's (N, m) device lens (FilterValues)
        cols = [evaluate_device(X, pc, s) for s in params.filters]
        F = torch.stack(cols, dim=1).contiguous() if len(cols) > 1 else cols[0].reshape(-1, 1)
    rng = torch.stack(torch.aminmax(F, dim=0), dim=1).cpu().numpy()
    cover = build_cover_from_range([(rng[a, 0], rng[a, 1]) for a in range(F.shape[1])],
                                   params.n, params.p)
    rows, offsets = eng.membership(F, cover)
    sizes = np.diff(offsets)
    budget = effective_mem_budget() if budget_bytes is None else budget_bytes
    orders = element_orders(sizes, params.strategy, budget)
    if rank == 0 and cancel_check is not None:
        cancel_check()
    costs = (element_costs(X, rows, offsets, sizes, params.eps, rank, world, dist)
             if balance == "kept" else np.asarray(sizes, dtype=np.float64) ** 2)
    big = big_elements(sizes, world, costs)
    parts = lpt_partition([0 if k in big else s for k, s in enumerate(sizes)], world, costs)
    mine = parts[rank]
    ranges, loc = pack_local(offsets, mine)
    st = np.zeros(8, dtype=np.int64)
    if mine and loc[-1] > 0:
        rows_loc = torch.cat([rows[a:b] for a, b in ranges])
        labels_loc, ncl_loc, st = cluster_device(
            X, rows_loc, loc, DbscanParams(params.eps, params.min_pts), orders[mine], None,
            engine)
    else:
        labels_loc = torch.empty(0, dtype=torch.int32, device=X.device)
        ncl_loc = np.zeros(len(mine), dtype=np.int32)
    if rank == 0 and cancel_check is not None:
        cancel_check()
    labels, ncl = gather_labels(labels_loc, ncl_loc, mine, parts, offsets, len(sizes), rank,
                                world, dist, X.device)
    for k in big:  # every rank takes an equal tile area of each big element
        a, b = int(offsets[k]), int(offsets[k + 1])
        with eng.BigElement(X, rows[a:b], params.eps, params.min_pts, int(orders[k]),
                            engine) as be:
            cap = device_window_tiles(X.device, X.shape[1], be.padded)
            lab_k, ncl_k = rowblock_cluster(be, rank, world, dist, cap, eng.merge_forest)
            st = st + be.stats()
        if rank == 0:
            labels[a:b] = lab_k
            ncl[k] = ncl_k
    if rank != 0:
        return None, st
    node_rows, node_off, n_nodes = eng.group_nodes(rows, offsets, labels, ncl)
    node_elem = np.repeat(np.arange(len(ncl)), ncl)
    edges = eng.nerve_edges(node_rows, node_off, n_nodes, X.shape[0])
    return DeviceGraph(F=F, cover=cover, sizes=sizes, orders=orders,
                       node_rows=node_rows, node_off=node_off, node_elem=node_elem,
                       n_nodes=n_nodes, edges=edges, dev_stats=st, timings={}), st
