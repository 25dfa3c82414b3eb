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
