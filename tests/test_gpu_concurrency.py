"""GPU: concurrent calls from several host threads, each on its own CUDA
stream (server.py:187-191 runs compute_mapper concurrently for different
datasets), give the same results as sequential calls — no shared mutable
device state between calls (the pairwise-sum program is a kernel argument)."""

import threading

import numpy as np
import pytest

from oracle import mapper_oracle as O

pytestmark = pytest.mark.gpu


def _case(d, seed):
    X = O.gmm(2500, d, 4, 3.0, seed)
    eps = O.dist_quantile(X, 0.04, seed)
    rng = np.random.default_rng(seed)
    members = [np.sort(rng.choice(2500, s, replace=False)) for s in (2400, 900, 300)]
    return X, eps, members


def _run(X, eps, members, engine):
    import torch

    from paper_2011_03209_b200 import engine as eng
    from paper_2011_03209_b200.device import require_gpu, to_device_f64

    dev = require_gpu()
    offs = np.zeros(len(members) + 1, dtype=np.int64)
    np.cumsum([len(m) for m in members], out=offs[1:])
    rows = torch.from_numpy(np.concatenate(members).astype(np.int64)).to(dev)
    orders = np.array([O.ORDER_PAIRWISE, O.ORDER_SEQUENTIAL, O.ORDER_PAIRWISE], dtype=np.uint8)
    lab, ncl, _ = eng.cluster(to_device_f64(X, dev), rows, offs, eps, 5, orders, engine)
    return lab.cpu().numpy(), ncl.copy()


@pytest.mark.parametrize("engine", [2, 1])
def test_concurrent_threads_match_sequential(engine):
    import torch

    dims = [100, 200, 64, 256] if engine == 2 else [5, 9, 300, 130]
    cases = [_case(d, 30 + i) for i, d in enumerate(dims)]
    want = [_run(*c, engine) for c in cases]
    got = [None] * len(cases)
    errors = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    got[i] = _run(*cases[i], engine)
                s.synchronize()
        except Exception as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(len(cases))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for (a, na), (b, nb) in zip(want, got):
        assert np.array_equal(a, b) and np.array_equal(na, nb)


def test_concurrent_l2_lens_different_dims():
    """The lens kernels' pairwise programs (one per d) are kernel arguments:
    threads with different d on different streams stay bit-exact."""
    import torch

    from paper_2011_03209_b200 import engine as eng
    from paper_2011_03209_b200.device import require_gpu, to_device_f64

    dev = require_gpu()
    rng = np.random.default_rng(0)
    mats = [rng.standard_normal((20000, d)) for d in (3, 130, 257, 1000)]
    want = [O.lens(X, "l2-norm") for X in mats]
    got = [None] * len(mats)
    errors = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                Xd = to_device_f64(mats[i], dev)
                for _ in range(5):
                    got[i] = eng.lens(Xd, 1).cpu().numpy()
                s.synchronize()
        except Exception as e:
            errors.append(e)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(len(mats))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for a, b in zip(want, got):
        assert np.array_equal(a, b)
