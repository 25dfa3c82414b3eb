"""GPU: the sharded build (distributed.build_distributed) end to end with real
kernels — LPT element sharding plus the row-block split of an element holding
more than 1/world of the pair work — equals the single-process build.

Only one GPU is available here, so the ranks share cuda:0 and talk over gloo:
every collective runs on the host between kernel launches and no kernel waits
on another rank (the NCCL path differs only in the collective calls, which the
CPU gloo tests cover with world 2 and 3)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data():
    from oracle import mapper_oracle as O

    X = O.gmm(6000, 64, 6, 4.0, 77)
    # with 3 intervals the middle element holds 81% of the pair work: row-blocked
    return X, O.dist_quantile(X, 0.03, 3)


def _params(eps):
    from paper_2011_03209_b200 import DistanceStrategy, FilterSpec, MapperParams

    return MapperParams(filters=[FilterSpec(kind="l2-norm")], n=[3], p=[0.3], eps=eps,
                        min_pts=5, strategy=DistanceStrategy(threshold=10 ** 9))


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2011_03209_b200 import from_array
    from paper_2011_03209_b200.device import to_device_f64
    from paper_2011_03209_b200.distributed import big_elements, build_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        X, eps = _data()
        dev = torch.device("cuda", 0)
        g, st = build_distributed(to_device_f64(X, dev), from_array(X), _params(eps), rank, world,
                                  dist, 1 << 62, 0)
        if rank == 0:
            q.put(dict(rows=g.node_rows.cpu().numpy(), off=g.node_off.cpu().numpy(),
                       elem=np.asarray(g.node_elem), edges=np.asarray(g.edges),
                       big=big_elements(g.sizes, world)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_build_equals_single(world):
    import torch
    import torch.multiprocessing as mp

    from paper_2011_03209_b200 import from_array
    from paper_2011_03209_b200.device import require_gpu, to_device_f64
    from paper_2011_03209_b200.pipeline import build_device

    X, eps = _data()
    dev = require_gpu()
    ref = build_device(to_device_f64(X, dev), from_array(X), _params(eps), 1 << 62, None, 0)
    torch.cuda.synchronize()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(600)
    assert all(p.exitcode == 0 for p in procs)
    assert got["big"], "the workload must exercise the row-block path"
    assert np.array_equal(got["rows"], ref.node_rows.cpu().numpy())
    assert np.array_equal(got["off"], ref.node_off.cpu().numpy())
    assert np.array_equal(got["elem"], np.asarray(ref.node_elem))
    assert np.array_equal(got["edges"], np.asarray(ref.edges))
