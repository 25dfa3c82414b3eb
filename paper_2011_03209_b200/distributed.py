"""Multi-GPU Mapper build: cover elements sharded across ranks (one process
per GPU, torch.distributed over NCCL), cluster memberships gathered to rank 0.

This replaces the reference's only parallelism strategy, the fork pool over
cover elements (clustering.py:281-315): elements are independent DBSCAN
instances, so the work partitions with no data-path collective; the single
exchange is the gather of per-entry cluster labels to the rank that builds
nodes and edges.

Every rank holds X and evaluates the (cheap, HBM-bound) lens and cover
itself, so memberships are identical on all ranks without communication.
Elements are assigned by LPT on the pair work n_k^2 (largest first onto the
least-loaded rank), a pure function of the sizes, so the assignment — and the
output — does not depend on the number of ranks or on timing.
"""

from __future__ import annotations

import heapq

import numpy as np


def lpt_partition(sizes, world: int) -> list:
    """Element ids per rank, largest n_k^2 first onto the least-loaded rank."""
    loads = [(0.0, r) for r in range(world)]
    heapq.heapify(loads)
    parts = [[] for _ in range(world)]
    order = sorted(range(len(sizes)), key=lambda k: (-int(sizes[k]) ** 2, k))
    for k in order:
        if int(sizes[k]) == 0:
            continue
        load, r = heapq.heappop(loads)
        parts[r].append(k)
        heapq.heappush(loads, (load + float(sizes[k]) ** 2, r))
    return [sorted(p) for p in parts]


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

    Collective: one all_gather of a fixed-size int32 buffer per rank (labels
    padded to the largest rank, cluster counts appended)."""
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
    out = torch.empty((world, cap), dtype=torch.int32, device=device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, buf)
    else:  # gloo (CPU tests of the host logic)
        chunks = list(out.unbind(0))
        dist.all_gather(chunks, buf)
        out = torch.stack(chunks)
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


def build_distributed(X, pc, params, rank: int, world: int, dist, budget_bytes=None,
                      engine: int = 0):
    """Sharded hot path. Returns a DeviceGraph on rank 0 and None elsewhere."""
    import torch

    from . import engine as eng
    from .clustering import DbscanParams, cluster_device, effective_mem_budget, element_orders
    from .cover import build_cover
    from .filters import FilterValues, evaluate_device
    from .pipeline import DeviceGraph

    cols = [evaluate_device(X, pc, s) for s in params.filters]
    F = torch.stack(cols, dim=1).contiguous() if len(cols) > 1 else cols[0].reshape(-1, 1)
    fv_host = F.cpu().numpy()
    cover = build_cover(FilterValues(values=fv_host.copy(), specs=list(params.filters)),
                        params.n, params.p)
    rows, offsets = eng.membership(F, cover)
    sizes = np.diff(offsets)
    budget = effective_mem_budget() if budget_bytes is None else budget_bytes
    orders = element_orders(sizes, params.strategy, budget)
    parts = lpt_partition(sizes, world)
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
    labels, ncl = gather_labels(labels_loc, ncl_loc, mine, parts, offsets, len(sizes), rank,
                                world, dist, X.device)
    if rank != 0:
        return None, st
    node_rows, node_off, n_nodes = eng.group_nodes(rows, offsets, labels, ncl)
    node_elem = np.repeat(np.arange(len(ncl)), ncl)
    edges = eng.nerve_edges(node_rows, node_off, n_nodes, X.shape[0])
    return DeviceGraph(F=F, fv_host=fv_host, cover=cover, sizes=sizes, orders=orders,
                       node_rows=node_rows, node_off=node_off, node_elem=node_elem,
                       n_nodes=n_nodes, edges=edges, dev_stats=st, timings={}), st
