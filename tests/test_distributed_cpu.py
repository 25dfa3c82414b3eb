"""CPU (gloo, world_size 2): host logic of the multi-GPU path — LPT element
partition and the label gather that rebuilds rank 0's per-entry labels."""

import os
import socket

import numpy as np
import pytest

from paper_2011_03209_b200.distributed import gather_labels, lpt_partition, pack_local


def test_lpt_partition_covers_every_nonempty_element_once():
    sizes = [5, 0, 100, 7, 7, 60, 1, 0, 33]
    for world in (1, 2, 3, 8):
        parts = lpt_partition(sizes, world)
        flat = sorted(k for p in parts for k in p)
        assert flat == [k for k, s in enumerate(sizes) if s]
        assert all(p == sorted(p) for p in parts)
    assert lpt_partition(sizes, 2) == lpt_partition(sizes, 2)  # deterministic


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        sizes = [13, 0, 40, 7, 22, 5]
        offsets = np.zeros(len(sizes) + 1, dtype=np.int64)
        np.cumsum(sizes, out=offsets[1:])
        truth = rng.integers(-1, 4, int(offsets[-1])).astype(np.int32)
        ncl_truth = np.array([int(truth[offsets[k]:offsets[k + 1]].max(initial=-1)) + 1
                              for k in range(len(sizes))], dtype=np.int32)
        parts = lpt_partition(sizes, world)
        mine = parts[rank]
        ranges, loc = pack_local(offsets, mine)
        lab_loc = torch.from_numpy(np.concatenate([truth[a:b] for a, b in ranges])
                                   if ranges else np.zeros(0, np.int32))
        full, ncl = gather_labels(lab_loc, ncl_truth[mine], mine, parts, offsets, len(sizes),
                                  rank, world, dist, torch.device("cpu"))
        if rank == 0:
            q.put((full.numpy().tolist() == truth.tolist(),
                   [int(x) for x in ncl] == ncl_truth.tolist()))
    finally:
        dist.destroy_process_group()


def test_gather_labels_gloo_world2():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    ok_labels, ok_ncl = q.get(timeout=5)
    assert ok_labels and ok_ncl


# ---------------------------------------------------------------------------
# row-block protocol for one huge element: host logic over gloo
# with a numpy model of the per-rank device steps (bm_big_* semantics)
# ---------------------------------------------------------------------------
from paper_2011_03209_b200.distributed import (area_windows, big_elements, rowblock_cluster,
                                               split_window, tri_rows)

_INT_MAX = 0x7FFFFFFF


def test_area_windows_partition_tile_rows():
    for T in (1, 2, 5, 37, 300):
        for world in (1, 2, 3, 8):
            w = area_windows(T, world)
            assert len(w) == world and w[0][0] == 0 and w[-1][1] == T
            assert all(w[r][1] == w[r + 1][0] for r in range(world - 1))
            areas = [tri_rows(T, b) - tri_rows(T, a) for a, b in w]
            if T >= 4 * world:  # balanced within one tile row of area
                assert max(areas) - min(areas) <= T
            for a, b in w:
                for cap in (1, 7, 10**9):
                    sub = split_window(a, b, T, cap)
                    assert [x for s in sub for x in range(*s)] == list(range(a, b))
                    assert all(tri_rows(T, e) - tri_rows(T, s) <= cap or e == s + 1
                               for s, e in sub)


def test_big_elements_rule():
    assert big_elements([10, 10, 10], 1) == []
    assert big_elements([100, 10, 10], 2) == [0]
    assert big_elements([10, 10, 10, 10], 2) == []


class _NumpyBig:
    """Model of engine.BigElement: the same window/count/union/border rules
    on a dense boolean eps-matrix (tile = 128 rows)."""

    TILE = 128

    def __init__(self, adj: np.ndarray, min_pts: int):
        import torch

        self.torch = torch
        self.n = adj.shape[0]
        self.tiles = -(-self.n // self.TILE)
        self.padded = self.tiles * self.TILE
        A = np.zeros((self.padded, self.padded), dtype=bool)
        A[: self.n, : self.n] = adj
        self.A = A
        self.min_pts = min_pts

    def zeros(self):
        return self.torch.zeros(self.padded, dtype=self.torch.int32)

    def _blocks(self, I0, I1):
        t = self.TILE
        for I in range(I0, I1):
            for J in range(I, self.tiles):
                yield I, J, slice(I * t, I * t + t), slice(J * t, J * t + t)

    def counts(self, I0, I1, cnt):
        c = cnt.numpy()
        for I, J, rs, cs in self._blocks(I0, I1):
            b = self.A[rs, cs]
            c[rs] += b.sum(1).astype(np.int32)
            if I != J:
                c[cs] += b.sum(0).astype(np.int32)

    def init(self, cnt, par, bmin):
        self.core = cnt.numpy() >= self.min_pts
        par.copy_(self.torch.arange(self.padded, dtype=self.torch.int32))
        bmin.fill_(_INT_MAX)

    @staticmethod
    def find(p, x):
        while p[x] != x:
            p[x] = p[p[x]]
            x = p[x]
        return x

    @classmethod
    def union(cls, p, a, b):
        a, b = cls.find(p, a), cls.find(p, b)
        if a != b:
            p[max(a, b)] = min(a, b)

    def components(self, I0, I1, par, bmin):
        p, bm, core = par.numpy(), bmin.numpy(), self.core
        for I, J, rs, cs in self._blocks(I0, I1):
            b = self.A[rs, cs]
            ri, cj = np.nonzero(b)
            ri = ri + rs.start
            cj = cj + cs.start
            for i, j in zip(ri, cj):
                if core[i] and core[j]:
                    self.union(p, int(i), int(j))
                elif core[j] and not core[i]:
                    bm[i] = min(bm[i], j)
                elif core[i] and not core[j] and I != J:
                    bm[j] = min(bm[j], i)

    def labels(self, par, bmin):
        p, bm, core = par.numpy(), bmin.numpy(), self.core
        root = np.full(self.n, -1)
        for i in range(self.n):
            if core[i]:
                root[i] = self.find(p, i)
            elif bm[i] != _INT_MAX:
                root[i] = self.find(p, int(bm[i]))
        first = {}
        for i in range(self.n):
            if root[i] >= 0 and root[i] not in first:
                first[root[i]] = i
        rank = {r: k for k, r in enumerate(sorted(first, key=first.get))}
        lab = np.array([rank[r] if r >= 0 else -1 for r in root], dtype=np.int32)
        return self.torch.from_numpy(lab), len(rank)


def _merge_forest_np(par, other):
    p, o = par.numpy(), other.numpy()
    for x in range(len(p)):
        if o[x] != x:
            _NumpyBig.union(p, x, int(o[x]))


def _rowblock_worker(rank, world, port, q, max_tiles):
    import torch.distributed as dist

    from oracle import mapper_oracle as orc

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X = orc.gmm(700, 4, 4, 3.0, seed=11)
        eps = orc.dist_quantile(X, 0.03)
        adj = orc.neighbour_matrix(X, eps, orc.ORDER_SEQUENTIAL)
        be = _NumpyBig(adj, 5)
        lab, ncl = rowblock_cluster(be, rank, world, dist, max_tiles, _merge_forest_np)
        if rank == 0:
            want = orc.dbscan_labels(adj, 5)
            q.put((lab.numpy().tolist() == want.tolist(), ncl == int(want.max()) + 1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,max_tiles", [(2, 10**9), (2, 3), (3, 2)])
def test_rowblock_protocol_gloo(world, max_tiles):
    pytest.importorskip("torch")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rowblock_worker, args=(r, world, port, q, max_tiles))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs)
    ok_labels, ok_ncl = q.get(timeout=5)
    assert ok_labels and ok_ncl
