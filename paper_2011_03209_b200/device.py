"""Device plumbing: which GPU, which stream, host<->device moves.

PyTorch owns every buffer (device tensors and pinned host staging); the C ABI
receives raw pointers plus the current torch stream. The GPU is chosen by the
B200MAP_DEVICE environment variable (default: torch's current device) — never
by DistanceStrategy.mode, which keeps nervemap's two modes only
(test_clustering.py:144 rejects a "gpu" mode).
"""

from __future__ import annotations

import os
import threading
import warnings

import numpy as np

from . import _native
from .errors import InternalError

try:  # torch is plumbing only; import lazily-failing for CPU-only tooling
    import torch
except Exception:  # pragma: no cover
    torch = None


def require_gpu():
    """Return the torch.device to run on; raise loudly when there is none."""
    if torch is None:
        raise InternalError("PyTorch is required for device memory management")
    if not torch.cuda.is_available():
        raise InternalError("no CUDA device: the B200 Mapper engine has no CPU fallback")
    _native.load()
    env = os.environ.get("B200MAP_DEVICE")
    if env is not None:
        dev = torch.device("cuda", int(env))
    else:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def stream_ptr(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


# ---------------------------------------------------------------------------
# Host -> device copies of pageable arrays through a reusable page-locked ring
# ---------------------------------------------------------------------------
STAGE_CHUNK = 64 << 20   # bytes per ring slot
STAGE_DEPTH = 4          # slots in flight
STAGE_MIN = 16 << 20     # smaller copies go straight through the driver


class _PinnedRing:
    """Per-device ring of page-locked chunks (allocated once, reused by every
    call): host threads fill slot i (parallel memcpy from the pageable
    source) while the copy engine drains slots i-1, i-2, ... to the device;
    a slot is refilled only after the event of its previous DMA."""

    def __init__(self, dev):
        self.dev = dev
        self.bufs = [torch.empty(STAGE_CHUNK, dtype=torch.uint8, pin_memory=True)
                     for _ in range(STAGE_DEPTH)]
        self.views = [b.numpy() for b in self.bufs]
        self.events = [None] * STAGE_DEPTH
        self.lock = threading.Lock()


_RINGS: dict = {}
_RINGS_LOCK = threading.Lock()
_POOL = None


def _copy_pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        n = int(os.environ.get("B200MAP_STAGE_THREADS", "16"))
        _POOL = ThreadPoolExecutor(max_workers=max(1, min(n, os.cpu_count() or 1)),
                                   thread_name_prefix="b200map-stage")
    return _POOL


def _ring(dev) -> _PinnedRing:
    key = (dev.type, dev.index)
    with _RINGS_LOCK:
        r = _RINGS.get(key)
        if r is None:
            r = _RINGS[key] = _PinnedRing(dev)
        return r


def _par_copy(dst: np.ndarray, src: np.ndarray):
    """memcpy of equal-size uint8 arrays on the staging threads (numpy drops
    the GIL inside the copy)."""
    pool = _copy_pool()
    n = src.size
    k = max(1, min(pool._max_workers, n >> 22))
    cuts = [i * n // k for i in range(k + 1)]
    list(pool.map(lambda i: np.copyto(dst[cuts[i]:cuts[i + 1]], src[cuts[i]:cuts[i + 1]]),
                  range(k)))


def h2d_into(dst, src: np.ndarray) -> None:
    """dst (contiguous device tensor) <- src (contiguous host array of the same
    byte size), on dst's current stream. Page-locked sources are copied
    directly; pageable ones are staged through the device's pinned ring."""
    nbytes = src.nbytes
    if nbytes == 0:
        return
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)  # read-only sources are only read
        t = torch.from_numpy(src)
    if t.is_pinned() or nbytes < STAGE_MIN:
        dst.copy_(t.view(dst.dtype).view(dst.shape), non_blocking=bool(t.is_pinned()))
        return
    ring = _ring(dst.device)
    stream = torch.cuda.current_stream(dst.device)
    s8 = src.reshape(-1).view(np.uint8)
    d8 = dst.view(-1).view(torch.uint8)
    with ring.lock:
        for i, off in enumerate(range(0, nbytes, STAGE_CHUNK)):
            m = min(STAGE_CHUNK, nbytes - off)
            slot = i % STAGE_DEPTH
            if ring.events[slot] is not None:
                ring.events[slot].synchronize()
            _par_copy(ring.views[slot][:m], s8[off:off + m])
            d8[off:off + m].copy_(ring.bufs[slot][:m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            ring.events[slot] = ev


def to_device_f64(arr: np.ndarray, dev):
    """Device copy of a host fp64 array: page-locked memory (e.g. the numpy
    view of a torch pin_memory() tensor) is copied asynchronously at full
    PCIe speed; pageable memory is staged through a reusable pinned ring
    (h2d_into) so the copy still streams at close to the link rate."""
    a = np.ascontiguousarray(arr, dtype=np.float64)
    out = torch.empty(a.shape, dtype=torch.float64, device=dev)
    h2d_into(out, a)
    return out


# ---------------------------------------------------------------------------
# Device-resident inputs across the library pieces (membership -> cluster_all
# -> build_graph): the reference's PointCloud.points / FilterValues.values are
# read-only by contract (dataset.py:66, filters.py:88), so the device copy of
# an object's array is kept with the object (by identity, dropped when the
# object is collected) instead of being uploaded by every call.
# ---------------------------------------------------------------------------
_DEV_CACHE: dict = {}
_DEV_CACHE_LOCK = threading.Lock()


def cached_device_array(owner, arr: np.ndarray, dev):
    """Device copy of `arr` (an array attribute of `owner`), cached while
    owner lives and the attribute still holds the same array buffer."""
    import weakref

    key = (id(owner), dev.index)
    with _DEV_CACHE_LOCK:
        hit = _DEV_CACHE.get(key)
        # the entry holds the host array itself: while cached it cannot be
        # freed, so `is` identifies it (no id/address reuse)
        if hit is not None and hit[0]() is owner and hit[1] is arr:
            return hit[2]
    t = to_device_f64(arr, dev)
    try:
        ref = weakref.ref(owner, lambda _r, k=key: _DEV_CACHE.pop(k, None))
    except TypeError:  # not weak-referenceable: no caching
        return t
    with _DEV_CACHE_LOCK:
        _DEV_CACHE[key] = (ref, arr, t)
    return t


def release_device_cache() -> None:
    """Drop every cached device copy and give the library's cached scratch
    (large buffers and the stream-ordered pool's reserve) back to the device,
    e.g. before handing the GPU to other work."""
    with _DEV_CACHE_LOCK:
        _DEV_CACHE.clear()
    from . import _native

    lib = _native.load()
    _native.check(lib.bm_release_scratch(), "release scratch")


def to_device_i64(arr: np.ndarray, dev):
    a = np.ascontiguousarray(arr, dtype=np.int64)
    return torch.from_numpy(a).to(dev)


def to_host(t) -> np.ndarray:
    return t.detach().to("cpu").numpy()
