"""GPU: the tensor-core (tcgen05 kind::i8) adjacency engine decides every eps
pair exactly like the fp64 engine (and hence like the reference)."""

import os

import numpy as np
import pytest

from oracle import mapper_oracle as O

pytestmark = pytest.mark.gpu


def labels(X, members, eps, min_pts, orders, engine):
    import torch

    from paper_2011_03209_b200 import engine as eng
    from paper_2011_03209_b200.device import require_gpu, to_device_f64

    dev = require_gpu()
    offs = np.zeros(len(members) + 1, dtype=np.int64)
    np.cumsum([len(m) for m in members], out=offs[1:])
    rows = torch.from_numpy(np.concatenate(members).astype(np.int64)).to(dev)
    lab, ncl, st = eng.cluster(to_device_f64(X, dev), rows, offs, eps, min_pts,
                               np.asarray(orders, dtype=np.uint8), engine)
    return lab.cpu().numpy(), ncl, st


@pytest.mark.parametrize("d", [32, 48, 64, 100, 128, 129, 200, 255, 256])
@pytest.mark.parametrize("q", [0.02, 0.15])
def test_tc_equals_exact(d, q):
    rng = np.random.default_rng(d)
    X = O.gmm(2500, d, 4, 3.0, d)
    eps = O.dist_quantile(X, q, d)
    members = [np.sort(rng.choice(2500, s, replace=False)) for s in (1, 130, 700, 2100)]
    for order in (O.ORDER_SEQUENTIAL, O.ORDER_PAIRWISE):
        orders = [order] * len(members)
        a, na, _ = labels(X, members, eps, 4, orders, 1)
        b, nb, st = labels(X, members, eps, 4, orders, 2)
        assert np.array_equal(a, b) and np.array_equal(na, nb), (d, q, order)


def test_tc_matches_oracle_cfg_like():
    X = O.gmm(4000, 256, 10, 5.0, 3)
    eps = 21.3
    rows = np.arange(4000)
    lab, ncl, st = labels(X, [rows], eps, 5, [O.ORDER_SEQUENTIAL], 2)
    clusters, noise = O.dbscan_element(X, rows, eps, 5, O.ORDER_SEQUENTIAL)
    got = [rows[lab == c].tolist() for c in range(int(ncl[0]))]
    assert got == clusters
    assert rows[lab < 0].tolist() == noise
    # the recheck handles a tiny fraction of the pairs
    assert st[1] < 0.01 * st[0]


def test_tc_exact_ties():
    import cases

    X, params = cases.tie_case()
    rows = np.arange(len(X))
    for order in (O.ORDER_SEQUENTIAL, O.ORDER_PAIRWISE):
        a, _, _ = labels(X, [rows], params["eps"], 2, [order], 1)
        b, _, _ = labels(X, [rows], params["eps"], 2, [order], 2)
        assert np.array_equal(a, b)


def test_tc_large_offsets_and_nan():
    rng = np.random.default_rng(1)
    X = O.gmm(600, 64, 3, 2.0, 1) + 1e6
    X[17, 5] = np.nan
    eps = O.dist_quantile(X[np.isfinite(X).all(axis=1)], 0.1)
    rows = np.arange(600)
    a, na, _ = labels(X, [rows], eps, 3, [0], 1)
    b, nb, _ = labels(X, [rows], eps, 3, [0], 2)
    assert np.array_equal(a, b) and np.array_equal(na, nb)
    assert a[17] == -1  # NaN point is in no neighbourhood (sqrt(NaN) <= eps is False)


@pytest.mark.parametrize("d", [16, 257])
def test_tc_dimension_range(d):
    """The tensor-core engine covers 32 <= d <= 256 (full-K B tiles in shared
    memory); asking for it outside raises DataError, the automatic engine
    takes the exact fp64 engine there."""
    from paper_2011_03209_b200.errors import DataError

    X = O.gmm(400, d, 3, 2.0, d)
    eps = O.dist_quantile(X, 0.1)
    rows = np.arange(400)
    with pytest.raises(DataError, match="tensor-core engine does not support"):
        labels(X, [rows], eps, 3, [0], 2)
    a, na, _ = labels(X, [rows], eps, 3, [0], 0)
    b, nb, _ = labels(X, [rows], eps, 3, [0], 1)
    assert np.array_equal(a, b) and np.array_equal(na, nb)


def test_tc_infinite_coordinates():
    """Rows with +-inf take the quantiser's clamping path (redone per row);
    they are in no neighbourhood, like NaN rows."""
    X = O.gmm(900, 96, 3, 2.0, 5)
    eps = O.dist_quantile(X, 0.1)
    X[3, 7] = np.inf
    X[400, 0] = -np.inf
    X[401, 95] = 1e300
    rows = np.arange(900)
    a, na, _ = labels(X, [rows], eps, 3, [0], 1)
    b, nb, _ = labels(X, [rows], eps, 3, [0], 2)
    assert np.array_equal(a, b) and np.array_equal(na, nb)
    assert a[3] == -1 and a[400] == -1


@pytest.mark.parametrize("qcap", ["40", "3"])
def test_recheck_queue_overflow_reruns(qcap):
    """A recheck queue too small for the undecided pairs is detected after the
    batch (no synchronisation inside it) and the batch reruns with a larger
    queue; windows (sync-checked) retry in place. Results are unchanged."""
    import subprocess
    import sys

    code = f"""
import os, sys, numpy as np
sys.path.insert(0, {repr(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))})
sys.path.insert(0, {repr(os.path.dirname(os.path.abspath(__file__)))})
from test_gpu_tc import labels
from oracle import mapper_oracle as O
X = O.gmm(3000, 128, 4, 3.0, 5)
eps = O.dist_quantile(X, 0.05, 5)
rows = np.arange(3000)
lab, ncl, st = labels(X, [rows], eps, 5, [O.ORDER_SEQUENTIAL], 2)
clusters, noise = O.dbscan_element(X, rows, eps, 5, O.ORDER_SEQUENTIAL)
got = [rows[lab == c].tolist() for c in range(int(ncl[0]))]
assert got == clusters and rows[lab < 0].tolist() == noise
print("rechecks", st[1])
"""
    for window in (None, "3"):
        env = dict(os.environ, B200MAP_TEST_QCAP=qcap)
        if window:
            env["B200MAP_WINDOW_TILES"] = window
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        assert int(r.stdout.split()[-1]) > int(qcap)  # the queue did overflow


@pytest.mark.parametrize("d", [32, 48, 64, 200, 256])
def test_direct_rows_equal_gathered_copy(monkeypatch, d):
    """The tensor-core engine reading X through the membership (int8 direction
    bound on the limb planes; default for even d) equals the engine on the
    gathered fp64 copy (fp32 direction bound; B200MAP_NO_DIRECT=1) and the
    oracle, with pruning on, grouped elements and NaN/inf rows."""
    X = O.gmm(3000, d, 6, 3.0, 40 + d)
    X[[5, 1700]] = np.nan
    X[[42], 3] = np.inf
    eps = O.dist_quantile(X[np.isfinite(X).all(axis=1)], 0.04, 2)
    rows = np.arange(3000)
    want = O.dbscan_labels(O.neighbour_matrix(X, eps, O.ORDER_SEQUENTIAL), 5)
    lab, _, _ = labels(X, [rows], eps, 5, [O.ORDER_SEQUENTIAL], 2)
    monkeypatch.setenv("B200MAP_NO_DIRECT", "1")
    lab_g, _, _ = labels(X, [rows], eps, 5, [O.ORDER_SEQUENTIAL], 2)
    assert lab.tolist() == want.tolist() == lab_g.tolist()
