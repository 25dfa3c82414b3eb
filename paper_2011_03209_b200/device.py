"""Device plumbing: which GPU, which stream, host<->device moves.

PyTorch owns every buffer (device tensors and pinned host staging); the C ABI
receives raw pointers plus the current torch stream. The GPU is chosen by the
B200MAP_DEVICE environment variable (default: torch's current device) — never
by DistanceStrategy.mode, which keeps nervemap's two modes only
(test_clustering.py:144 rejects a "gpu" mode).
"""

from __future__ import annotations

import os
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


def to_device_f64(arr: np.ndarray, dev):
    """Device copy of a host fp64 array. Page-locked host memory (e.g. the
    numpy view of a torch pin_memory() tensor) is copied asynchronously at
    full PCIe speed; pageable memory goes through the driver's staged copy
    (pinning it first would cost a fresh page-locked allocation per call)."""
    a = np.ascontiguousarray(arr, dtype=np.float64)
    with warnings.catch_warnings():
        # read-only PointCloud arrays: torch only reads them (H2D source)
        warnings.simplefilter("ignore", UserWarning)
        t = torch.from_numpy(a)
    return t.to(dev, non_blocking=bool(a.nbytes and t.is_pinned()))


def to_device_i64(arr: np.ndarray, dev):
    a = np.ascontiguousarray(arr, dtype=np.int64)
    return torch.from_numpy(a).to(dev)


def to_host(t) -> np.ndarray:
    return t.detach().to("cpu").numpy()
