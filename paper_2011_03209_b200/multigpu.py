"""Several GPUs behind the drop-in API: compute_mapper drives N devices from
one process when B200MAP_GPUS / B200MAP_DEVICES asks for it.

The reference's only parallelism knob is `threads` on compute_mapper /
cluster_all, a fork pool over cover elements (clustering.py:238-242,
281-315). `threads` keeps its meaning here (validated, never forks); the GPU
count is a separate knob:

  B200MAP_GPUS=N          the first N visible devices ("all": every one)
  B200MAP_DEVICES=0,1,..  an explicit device list (a device may repeat:
                          "0,0,0" runs the 3-device protocol on one GPU —
                          the GPU tests use it; ranks never wait on each
                          other inside a kernel, only at host barriers)

One host thread per device runs the SPMD program of distributed.py
(build_distributed: lens/cover on every device, elements by LPT, one huge
element by row blocks, labels gathered to device 0) with ThreadGroup as its
collective layer: the collectives are peer copies between the devices' HBM
(cudaMemcpyPeerAsync over NVLink/NVSwitch through torch's cross-device
copy) between host barriers, the same contract as torch.distributed's
(all_reduce SUM/MIN, all_gather_into_tensor, gather). Under torchrun the
same program runs with the NCCL process group instead (bench.py --gpus N).

X reaches the devices sharded: device r copies rows
[r*B, (r+1)*B) from the host over its own PCIe link, then an all-gather over
NVLink completes every device's replica, so the H2D time falls ~1/N.
"""

from __future__ import annotations

import os
import threading

import numpy as np

from .errors import DataError, InternalError

GPUS_ENV = "B200MAP_GPUS"
DEVICES_ENV = "B200MAP_DEVICES"


def gpu_devices() -> list:
    """Device indices the drop-in API should drive (one entry per rank)."""
    import torch

    raw = os.environ.get(DEVICES_ENV)
    if raw:
        try:
            devs = [int(x) for x in raw.split(",") if x.strip()]
        except ValueError:
            raise DataError(f"{DEVICES_ENV} must be a comma list of device ids") from None
        n = torch.cuda.device_count()
        if not devs or any(d < 0 or d >= n for d in devs):
            raise DataError(f"{DEVICES_ENV}={raw!r}: only {n} device(s) visible")
        return devs
    raw = os.environ.get(GPUS_ENV)
    if raw:
        n = torch.cuda.device_count()
        if raw == "all":
            return list(range(n))
        try:
            k = int(raw)
        except ValueError:
            raise DataError(f"{GPUS_ENV} must be an integer or 'all'") from None
        if not 1 <= k <= n:
            raise DataError(f"{GPUS_ENV}={k}: {n} device(s) visible")
        return list(range(k))
    return []


class ThreadGroup:
    """In-process collectives over per-device tensors, one host thread per
    rank. Each call is a rendezvous: every rank's stream is drained, the
    tensors are published, each rank reads its peers' tensors with
    cross-device copies onto its own stream, and a second barrier keeps the
    published tensors alive until every reader has copied them."""

    def __init__(self, world: int):
        import torch.distributed as tdist

        self.world = world
        self.ReduceOp = tdist.ReduceOp
        self._bar = threading.Barrier(world)
        self._slots = [None] * world

    def rank_view(self, rank: int) -> "RankView":
        return RankView(self, rank)

    def abort(self):
        self._bar.abort()

    # ---- internals (called through RankView)
    def _publish(self, rank, t):
        import torch

        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()
        self._slots[rank] = t
        self._bar.wait()

    def _done(self, t):
        import torch

        if t is not None and t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()
        self._bar.wait()


class RankView:
    """The torch.distributed surface distributed.py uses, for one rank."""

    def __init__(self, group: ThreadGroup, rank: int):
        self.g = group
        self.rank = rank
        self.ReduceOp = group.ReduceOp

    def get_backend(self):
        return "threads"

    def get_rank(self):
        return self.rank

    def get_world_size(self):
        return self.g.world

    def barrier(self):
        self.g._bar.wait()

    def all_reduce(self, t, op=None):
        import torch

        g = self.g
        op = g.ReduceOp.SUM if op is None else op
        g._publish(self.rank, t)
        others = []
        for r in range(g.world):
            if r != self.rank:  # always a copy (.to() aliases on the same device)
                o = torch.empty_like(t)
                o.copy_(g._slots[r], non_blocking=True)
                others.append(o)
        g._done(t)  # every rank holds its peers' copies: t may now change
        for o in others:
            if op == g.ReduceOp.SUM:
                t.add_(o)
            elif op == g.ReduceOp.MIN:
                t.copy_(t.minimum(o))
            elif op == g.ReduceOp.MAX:
                t.copy_(t.maximum(o))
            else:
                raise InternalError(f"ThreadGroup: unsupported reduce op {op}")
        g._done(t)

    def all_gather_into_tensor(self, out, t):
        g = self.g
        g._publish(self.rank, t)
        n = t.numel()
        flat = out.view(-1)
        for r in range(g.world):
            src = g._slots[r].reshape(-1)
            dst = flat[r * n:(r + 1) * n]
            if src.data_ptr() != dst.data_ptr() or src.device != dst.device:
                dst.copy_(src, non_blocking=True)
        g._done(out)

    def all_gather(self, chunks, t):
        g = self.g
        g._publish(self.rank, t)
        for r in range(g.world):
            chunks[r].copy_(g._slots[r], non_blocking=True)
        g._done(chunks[0])

    def gather(self, t, gather_list=None, dst=0):
        g = self.g
        g._publish(self.rank, t)
        if self.rank == dst:
            for r in range(g.world):
                gather_list[r].copy_(g._slots[r], non_blocking=True)
        g._done(gather_list[0] if self.rank == dst else None)


def upload_sharded(Xh, rank: int, world: int, dist, device):
    """rank r copies its 1/world of X's rows host -> device over
    its own PCIe link, then one all-gather (NVLink) fills every replica.
    Xh: host fp64 array/tensor (page-locked for full PCIe speed). Returns the
    (N, d) device tensor (a view of an (Npad, d) buffer; pad rows are zero)."""
    import torch

    n, d = Xh.shape
    B = -(-n // world)
    buf = torch.empty((B * world, d), dtype=torch.float64, device=device)
    a, b = min(rank * B, n), min((rank + 1) * B, n)
    mine = buf[rank * B:(rank + 1) * B]
    if b > a:
        if isinstance(Xh, torch.Tensor):
            mine[: b - a].copy_(Xh[a:b], non_blocking=bool(Xh.is_pinned()))
        elif buf.is_cuda:
            from .device import h2d_into

            h2d_into(mine[: b - a], np.ascontiguousarray(Xh[a:b]))
        else:
            mine[: b - a].copy_(torch.from_numpy(np.ascontiguousarray(Xh[a:b])))
    if b - a < B:
        mine[b - a:].zero_()
    if world > 1:
        if dist.get_backend() in ("nccl", "threads"):
            dist.all_gather_into_tensor(buf, mine)
        else:  # gloo (CPU tests)
            chunks = list(buf.view(world, B, d).unbind(0))
            dist.all_gather(chunks, mine.clone())
    return buf[:n]


def run_ranks(devices: list, fn):
    """Run fn(rank, world, view, device) on one host thread per device;
    returns the per-rank results (the first exception is re-raised after
    every thread has stopped; a failing rank aborts the others' barriers)."""
    import torch

    world = len(devices)
    group = ThreadGroup(world)
    results = [None] * world
    errors = [None] * world

    def body(r):
        try:
            dev = torch.device("cuda", devices[r])
            torch.cuda.set_device(dev)
            with torch.cuda.device(dev):
                results[r] = fn(r, world, group.rank_view(r), dev)
                torch.cuda.current_stream(dev).synchronize()
        except BaseException as e:  # noqa: BLE001 - propagate any rank's failure
            errors[r] = e
            group.abort()

    threads = [threading.Thread(target=body, args=(r,), name=f"b200map-rank{r}")
               for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    first = next((e for e in errors if e is not None and
                  not isinstance(e, threading.BrokenBarrierError)), None)
    if first is None:
        first = next((e for e in errors if e is not None), None)
    if first is not None:
        raise first
    return results
