"""GPU: host inputs — pageable arrays staged through the pinned ring
(device.h2d_into), concurrent stagers on one device, and the device-resident
copy of a PointCloud / FilterValues reused across the library pieces."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nbytes", [8, 1 << 20, (16 << 20) + 8, (64 << 20) * 3 + 4096 * 8 + 8])
def test_h2d_ring_roundtrip(nbytes):
    import torch

    from paper_2011_03209_b200.device import h2d_into, require_gpu

    dev = require_gpu()
    n = nbytes // 8
    src = np.random.default_rng(n).standard_normal(n)
    dst = torch.empty(n, dtype=torch.float64, device=dev)
    h2d_into(dst, src)
    src[:] = -1.0  # the staging copy is complete on return: the source may change
    torch.cuda.synchronize()
    assert np.array_equal(dst.cpu().numpy(), np.random.default_rng(n).standard_normal(n))


def test_h2d_ring_concurrent_threads():
    import torch

    from paper_2011_03209_b200.device import require_gpu, to_device_f64

    dev = require_gpu()
    arrays = [np.random.default_rng(s).standard_normal((1 << 21) + s) for s in range(4)]
    out = [None] * 4

    def work(i):
        with torch.cuda.device(dev):
            t = to_device_f64(arrays[i], dev)
            torch.cuda.current_stream(dev).synchronize()
            out[i] = t.cpu().numpy()

    ts = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for a, o in zip(arrays, out):
        assert np.array_equal(a, o)


def test_library_pieces_upload_points_once(monkeypatch):
    """membership -> cluster_all -> build_graph on one PointCloud and one
    FilterValues uploads each array once (the reference's inputs are
    read-only; device.cached_device_array)."""
    from paper_2011_03209_b200 import (DbscanParams, DistanceStrategy, FilterSpec, FilterValues,
                                       build_cover, build_graph, cluster_all, device, from_array,
                                       membership)
    from oracle import mapper_oracle as O

    X = O.gmm(20000, 64, 8, 4.0, 9)
    F = np.column_stack([O.lens(X, "l2-norm"), X[:, 0]])
    calls = []
    real = device.to_device_f64

    def counting(arr, dev):
        calls.append(arr.shape)
        return real(arr, dev)

    monkeypatch.setattr(device, "to_device_f64", counting)
    pc = from_array(X)
    fv = FilterValues(values=F, specs=[FilterSpec(kind="l2-norm")] * 2)
    cover = build_cover(fv, [4, 3], [0.3, 0.2])
    members = membership(fv, cover)
    eps = O.dist_quantile(X, 0.03)
    cl = cluster_all(pc, members, DbscanParams(eps, 5), DistanceStrategy())
    g = build_graph(cl, pc, fv, cover, manifest={})
    assert g.n_nodes > 0
    assert sorted(calls) == sorted([X.shape, F.shape])
    # a new object with the same contents uploads again
    cluster_all(from_array(X), members, DbscanParams(eps, 5), DistanceStrategy())
    assert calls.count(X.shape) == 2


def test_release_device_cache_then_rebuild(golden):
    """release_device_cache() drops the device copies and the library's cached
    scratch (large buffers + pool reserve); the next build allocates again and
    still gives the reference's bytes."""
    import torch

    import cases
    from paper_2011_03209_b200 import device
    from test_gpu_pipeline import graph_bytes

    X, p = cases.cfg1()
    z = golden("cfg1")
    assert graph_bytes(X, p, 0) == z["graph"].tobytes()
    torch.cuda.synchronize()
    device.release_device_cache()
    assert graph_bytes(X, p, 0) == z["graph"].tobytes()
