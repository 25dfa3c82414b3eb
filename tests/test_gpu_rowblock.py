"""GPU: the row-block path for a huge element.

(1) bm_cluster_elements with forced small row windows (B200MAP_WINDOW_TILES)
equals the one-window result and the oracle: two passes (counts, then
components with recomputed windows) change nothing.
(2) The bm_big_* per-rank steps, driven for several emulated ranks one after
another in ONE process (no kernel waits on another rank; the collectives are
done on the host between the steps exactly as distributed.rowblock_cluster
orders them), give the element's oracle labels for every world size."""

import numpy as np
import pytest

from oracle import mapper_oracle as O

pytestmark = pytest.mark.gpu


def _run(X, members, eps, min_pts, orders, engine):
    import torch

    from paper_2011_03209_b200 import engine as eng
    from paper_2011_03209_b200.device import require_gpu, to_device_f64

    dev = require_gpu()
    offs = np.zeros(len(members) + 1, dtype=np.int64)
    np.cumsum([len(m) for m in members], out=offs[1:])
    rows = torch.from_numpy(np.concatenate(members).astype(np.int64)).to(dev)
    lab, ncl, st = eng.cluster(to_device_f64(X, dev), rows, offs, eps, min_pts,
                               np.asarray(orders, dtype=np.uint8), engine)
    return lab.cpu().numpy(), ncl.copy(), st


@pytest.mark.parametrize("engine,d", [(2, 64), (2, 256), (1, 5)])
@pytest.mark.parametrize("cap", [1, 4, 13])
def test_forced_windows_equal_single_window(monkeypatch, engine, d, cap):
    X = O.gmm(3000, d, 5, 3.0, 40 + d)
    eps = O.dist_quantile(X, 0.05, 1)
    rng = np.random.default_rng(d)
    members = [np.sort(rng.choice(3000, s, replace=False)) for s in (2900, 40, 700)]
    orders = [O.ORDER_SEQUENTIAL, O.ORDER_PAIRWISE, O.ORDER_PAIRWISE]
    monkeypatch.delenv("B200MAP_WINDOW_TILES", raising=False)
    a, na, _ = _run(X, members, eps, 5, orders, engine)
    monkeypatch.setenv("B200MAP_WINDOW_TILES", str(cap))
    b, nb, st = _run(X, members, eps, 5, orders, engine)
    assert np.array_equal(a, b) and np.array_equal(na, nb)
    # and both equal the oracle
    pos = 0
    for m, o in zip(members, orders):
        clusters, noise = O.dbscan_element(X, m, eps, 5, o)
        lab = a[pos:pos + len(m)]
        assert [m[lab == c].tolist() for c in range(int(lab.max(initial=-1)) + 1)] == clusters
        assert m[lab < 0].tolist() == noise
        pos += len(m)


def _emulated_ranks(X, rows_np, eps, min_pts, order, world, max_tiles, engine=0):
    import torch

    from paper_2011_03209_b200 import engine as eng
    from paper_2011_03209_b200.device import require_gpu, to_device_f64
    from paper_2011_03209_b200.distributed import area_windows, split_window

    dev = require_gpu()
    Xd = to_device_f64(X, dev)
    rows = torch.from_numpy(rows_np.astype(np.int64)).to(dev)
    handles = [eng.BigElement(Xd, rows, eps, min_pts, order, engine) for _ in range(world)]
    try:
        T = handles[0].tiles
        wins = []
        for r in range(world):
            I0, I1 = area_windows(T, world)[r]
            wins.append(split_window(I0, I1, T, max_tiles) if I1 > I0 else [])
        cnts = []
        for r, be in enumerate(handles):
            c = be.zeros()
            for w in wins[r]:
                be.counts(w[0], w[1], c)
            cnts.append(c)
        cnt = torch.stack(cnts).sum(0).to(torch.int32)          # all_reduce(sum)
        pars, bmins = [], []
        for r, be in enumerate(handles):
            par, bmin = be.zeros(), be.zeros()
            be.init(cnt, par, bmin)
            for w in reversed(wins[r]):
                be.components(w[0], w[1], par, bmin)
            pars.append(par)
            bmins.append(bmin)
        bmin = torch.stack(bmins).min(0).values.contiguous()    # all_reduce(min)
        par = pars[0]
        for r in range(1, world):                                 # gather + merge on rank 0
            eng.merge_forest(par, pars[r])
        lab, ncl = handles[0].labels(par, bmin)
        return lab.cpu().numpy(), ncl, cnt.cpu().numpy()
    finally:
        for be in handles:
            be.close()


@pytest.mark.parametrize("world,max_tiles", [(1, 10**9), (2, 10**9), (3, 5), (8, 2)])
@pytest.mark.parametrize("engine,d", [(2, 128), (1, 7)])
def test_big_element_protocol_emulated(world, max_tiles, engine, d):
    X = O.gmm(2300, d, 4, 3.0, 7 + d)
    eps = O.dist_quantile(X, 0.04, 2)
    rows = np.arange(0, 2300, dtype=np.int64)
    lab, ncl, cnt = _emulated_ranks(X, rows, eps, 5, O.ORDER_SEQUENTIAL, world, max_tiles,
                                    engine)
    adj = O.neighbour_matrix(X[rows], eps, O.ORDER_SEQUENTIAL)
    # counts are per padded row (grouped order, pads 0): compare as multisets
    want_cnt = np.concatenate([adj.sum(1), np.zeros(len(cnt) - len(rows), dtype=np.int64)])
    assert np.array_equal(np.sort(cnt), np.sort(want_cnt))
    want = O.dbscan_labels(adj, 5)
    assert np.array_equal(lab, want)
    assert ncl == int(want.max(initial=-1)) + 1
