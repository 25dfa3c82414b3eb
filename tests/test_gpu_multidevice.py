"""GPU: compute_mapper on several devices from one process (multigpu.py:
B200MAP_DEVICES / B200MAP_GPUS), byte-identical to one device.

Only one GPU exists on the test box, so "0,0" / "0,0,0" run the 2- and
3-rank protocol with every rank on cuda:0 (each rank its own X replica,
sharded upload + all-gather, LPT by kept tile pairs, row blocks of a big
element by kept tiles, labels gathered to rank 0). Ranks meet only at host
barriers between kernels; no kernel waits on another rank."""

import hashlib

import numpy as np
import pytest

import cases
from test_gpu_pipeline import graph_bytes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("devices", ["0,0", "0,0,0"])
def test_cfg2_bytes_multi_device(golden, monkeypatch, devices):
    z = golden("cfg2")
    X, p = cases.cfg2()
    monkeypatch.setenv("B200MAP_DEVICES", devices)
    assert graph_bytes(X, p) == z["graph"].tobytes()


@pytest.mark.parametrize("devices", ["0,0", "0,0,0", "0,0,0,0,0,0,0,0"])
def test_near_eps_single_element_row_blocks(golden, monkeypatch, devices):
    """One element (the whole cloud) holds all the work: it is split into
    row blocks balanced on kept tile pairs, and the near-eps decisions still
    equal the reference's."""
    z = golden("near_eps")
    X, p = cases.near_eps_case()
    monkeypatch.setenv("B200MAP_DEVICES", devices)
    got = graph_bytes(X, dict(p, mode="precomputed"))
    assert hashlib.sha256(got).hexdigest() == str(z["pre_sha"])


@pytest.mark.parametrize("devices", ["0,0", "0,0,0"])
@pytest.mark.parametrize("seed", [0, 7, 19, 33, 48])
def test_instances_multi_device(golden, monkeypatch, devices, seed):
    z = golden("instances")
    X, p = cases.instance(seed)
    monkeypatch.setenv("B200MAP_DEVICES", devices)
    assert graph_bytes(X, p) == z[f"g{seed}"].tobytes()


def test_big_element_mixed_workload(monkeypatch):
    """3 intervals: the middle element holds most of the work (row blocks),
    the others go by LPT — equal to the single-device build."""
    from oracle import mapper_oracle as O

    X = O.gmm(6000, 64, 6, 4.0, 77)
    eps = O.dist_quantile(X, 0.03, 3)
    p = dict(filters=[{"kind": "l2-norm"}], n=[3], p=[0.3], eps=eps, min_pts=5, norm="none",
             mode="precomputed", threshold=10 ** 9)
    want = graph_bytes(X, p)
    for devices in ("0,0", "0,0,0", "0,0,0,0"):
        monkeypatch.setenv("B200MAP_DEVICES", devices)
        assert graph_bytes(X, p) == want, devices


def test_element_work_matches_engine_tiles():
    """bm_element_work's kept tile pairs are exactly the tile pairs the exact
    engine computes (same grouping and pruning)."""
    import torch

    from oracle import mapper_oracle as O
    from paper_2011_03209_b200 import engine as eng
    from paper_2011_03209_b200.device import require_gpu, to_device_f64

    X = O.gmm(20000, 64, 8, 4.0, 5)
    dev = require_gpu()
    Xd = to_device_f64(X, dev)
    f = O.lens(X, "l2-norm")
    members = O.membership(f[:, None], [O.cover_axis(f, 6, 0.3)])
    off = np.zeros(len(members) + 1, dtype=np.int64)
    np.cumsum([len(m) for m in members], out=off[1:])
    rows = torch.from_numpy(np.concatenate(members).astype(np.int64)).to(dev)
    eps = O.dist_quantile(X, 0.02)
    kept = eng.element_work(Xd, rows, off, eps)
    _, _, st = eng.cluster(Xd, rows, off, eps, 5, np.zeros(len(members), np.uint8), 1)
    assert int(kept.sum()) == int(st[3] - st[2])
    assert (kept > 0).all() and int(st[2]) > 0  # something was pruned


def test_cancel_check_aborts_every_rank(monkeypatch):
    from paper_2011_03209_b200 import compute_mapper, from_array

    from test_gpu_pipeline import params_of

    X, p = cases.cfg1()
    monkeypatch.setenv("B200MAP_DEVICES", "0,0,0")

    class Stop(Exception):
        pass

    def cancel():
        raise Stop()

    with pytest.raises(Stop):
        compute_mapper(from_array(X), params_of(p), cancel_check=cancel)
