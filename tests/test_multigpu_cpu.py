"""CPU: the in-process collective layer of the multi-device drop-in path
(multigpu.ThreadGroup: one host thread per rank) — its collectives, the
sharded upload of X and the row-block protocol of one huge
element running over it (the same distributed.py code NCCL ranks run)."""

import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2011_03209_b200.distributed import (kept_windows, lpt_partition,  # noqa: E402
                                               rowblock_cluster, split_window_kept)
from paper_2011_03209_b200.multigpu import ThreadGroup, upload_sharded  # noqa: E402


def run_threads(world, fn):
    g = ThreadGroup(world)
    out = [None] * world
    err = []

    def body(r):
        try:
            out[r] = fn(r, g.rank_view(r))
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            g.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(60)
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_collectives(world):
    def fn(r, dist):
        a = torch.arange(6, dtype=torch.int64) * (r + 1)
        dist.all_reduce(a, op=dist.ReduceOp.SUM)
        b = torch.full((4,), 10 - r, dtype=torch.int32)
        dist.all_reduce(b, op=dist.ReduceOp.MIN)
        out = torch.empty(world * 3, dtype=torch.int32)
        dist.all_gather_into_tensor(out, torch.full((3,), r, dtype=torch.int32))
        gl = [torch.empty(2, dtype=torch.int64) for _ in range(world)] if r == 0 else None
        dist.gather(torch.tensor([r, -r]), gl, dst=0)
        return a.tolist(), b.tolist(), out.tolist(), [x.tolist() for x in gl] if gl else None

    res = run_threads(world, fn)
    tot = sum(range(1, world + 1))
    for r, (a, b, out, gl) in enumerate(res):
        assert a == [i * tot for i in range(6)]
        assert b == [10 - (world - 1)] * 4
        assert out == [q for q in range(world) for _ in range(3)]
        if r == 0:
            assert gl == [[q, -q] for q in range(world)]


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_upload_sharded_replicates_rows(world):
    X = np.random.default_rng(world).standard_normal((1003, 7))

    def fn(r, dist):
        return upload_sharded(X, r, world, dist, torch.device("cpu")).numpy().copy()

    for got in run_threads(world, fn):
        assert np.array_equal(got, X)


def test_kept_windows_balance_and_cover():
    rng = np.random.default_rng(3)
    for T in (1, 3, 40, 200):
        kept = rng.integers(0, 50, T)
        rf = np.concatenate([[0], np.cumsum(kept)])
        for world in (1, 2, 3, 8):
            w = kept_windows(rf, world)
            assert w[0][0] == 0 and w[-1][1] == T and len(w) == world
            assert all(w[i][1] == w[i + 1][0] for i in range(world - 1))
            if T >= 8 * world:
                share = [rf[b] - rf[a] for a, b in w]
                assert max(share) - rf[-1] / world <= kept.max() + 1
            for a, b in w:
                for cap in (1, 30, 10 ** 9):
                    sub = split_window_kept(a, b, rf, cap)
                    assert [x for s in sub for x in range(*s)] == list(range(a, b))
                    assert all(rf[e] - rf[s] <= cap or e == s + 1 for s, e in sub)


def test_lpt_with_costs():
    sizes = [10, 10, 10, 10]
    assert lpt_partition(sizes, 2, costs=[100, 1, 1, 98]) == [[0], [1, 2, 3]]
    assert lpt_partition(sizes, 2) == [[0, 2], [1, 3]]  # n_k^2: all equal


@pytest.mark.parametrize("world,max_tiles", [(2, 10 ** 9), (3, 2), (4, 5)])
def test_rowblock_protocol_over_threads(world, max_tiles):
    """The row-block protocol of distributed.py over ThreadGroup, with the
    numpy model of the per-rank device steps, equals the oracle's DBSCAN."""
    from oracle import mapper_oracle as orc
    from test_distributed_cpu import _merge_forest_np, _NumpyBig

    X = orc.gmm(900, 4, 4, 3.0, seed=12)
    eps = orc.dist_quantile(X, 0.03)
    adj = orc.neighbour_matrix(X, eps, orc.ORDER_SEQUENTIAL)
    want = orc.dbscan_labels(adj, 5)

    class KeptModel(_NumpyBig):  # kept-tile windows (every tile pair kept)
        def row_tiles(self):
            T = self.tiles
            return np.concatenate([[0], np.cumsum([T - I for I in range(T)])])

    def fn(r, dist):
        be = KeptModel(adj, 5)
        return rowblock_cluster(be, r, world, dist, max_tiles, _merge_forest_np)

    lab, ncl = run_threads(world, fn)[0]
    assert lab.numpy().tolist() == want.tolist() and ncl == int(want.max()) + 1
