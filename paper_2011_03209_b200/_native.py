"""ctypes binding of libb200map.so (the C ABI declared in include/b200map.h).

This is the only module that touches the shared library. Every wrapper maps
the ABI status to the package's exception taxonomy (errors.py, mirroring
nervemap/errors.py:9-17): BM_ERR_DATA -> DataError, anything else ->
InternalError. There is no CPU fallback: if the library or a CUDA device is
missing, the hot-path entry points raise InternalError.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DataError, InternalError

_LIB_NAME = "libb200map.so"
_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, _LIB_NAME)

BM_OK = 0
BM_ERR_DATA = -1
BM_ERR_INTERNAL = -2
BM_ERR_NOMEM = -3

ORDER_SEQUENTIAL = 0
ORDER_PAIRWISE = 1

LENS_COLUMN = 0
LENS_L2 = 1
LENS_LINF = 2

PLENS_ECC_MEAN = 0
PLENS_ECC_RMS = 1
PLENS_ECC_POW = 2
PLENS_ECC_MAX = 3
PLENS_DENSITY = 4
PLENS_NN_MIN = 5

ENGINE_AUTO = 0
ENGINE_EXACT = 1
ENGINE_TC = 2

# symbol -> (restype, argtypes); must match include/b200map.h exactly
_c_i64 = ctypes.c_int64
_c_i32 = ctypes.c_int32
_vp = ctypes.c_void_p
_SIGNATURES = {
    "bm_abi_version": (ctypes.c_int, []),
    "bm_last_error": (ctypes.c_char_p, []),
    "bm_launch_count": (ctypes.c_int64, []),
    "bm_release_scratch": (ctypes.c_int, []),
    "bm_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "bm_device_free_bytes": (ctypes.c_int, [_vp]),
    "bm_lens_f64": (ctypes.c_int, [ctypes.c_int, _vp, _c_i64, _c_i64, _c_i64, _vp, _vp]),
    "bm_pairwise_lens": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, _vp, _c_i64, _c_i64, _vp,
                                        _c_i64, _vp, _c_i64, _vp, _vp]),
    "bm_normalize_f64": (ctypes.c_int, [ctypes.c_int, _vp, _c_i64, _c_i64, _vp, _vp]),
    "bm_membership_count": (ctypes.c_int, [_vp, _c_i64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp]),
    "bm_membership_fill": (ctypes.c_int, [_vp, _c_i64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bm_cluster_elements": (ctypes.c_int, [_vp, _c_i64, _c_i64, _vp, _vp, _c_i64, ctypes.c_double,
                                           _c_i32, _vp, ctypes.c_int, _vp, _vp, _vp, _vp]),
    "bm_pairwise_distances": (ctypes.c_int, [_vp, _c_i64, _c_i64, _vp, _c_i64, ctypes.c_int, _vp, _vp]),
    "bm_big_open": (ctypes.c_int, [_vp, _c_i64, _c_i64, _vp, _c_i64, ctypes.c_double, _c_i32,
                                   ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "bm_big_counts": (ctypes.c_int, [_vp, _c_i32, _c_i32, _vp]),
    "bm_big_init": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "bm_big_components": (ctypes.c_int, [_vp, _c_i32, _c_i32, _vp, _vp]),
    "bm_big_labels": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "bm_big_stats": (ctypes.c_int, [_vp, _vp]),
    "bm_big_row_tiles": (ctypes.c_int, [_vp, _vp]),
    "bm_big_close": (ctypes.c_int, [_vp]),
    "bm_element_work": (ctypes.c_int, [_vp, _c_i64, _c_i64, _vp, _vp, _c_i64, ctypes.c_double,
                                       _vp, _vp]),
    "bm_merge_forest": (ctypes.c_int, [_vp, _vp, _c_i64, _vp]),
    "bm_group_nodes": (ctypes.c_int, [_vp, _vp, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bm_nerve_edges": (ctypes.c_int, [_vp, _vp, _c_i64, _c_i64, _vp, _vp, _vp]),
    "bm_json_nodes": (ctypes.c_int, [_c_i64, _vp, _vp, _vp, _vp, _c_i64, _vp, _vp, _vp, _vp,
                                     _c_i32, _vp, _vp, _vp, _c_i64, _vp]),
    "bm_node_stats": (ctypes.c_int, [_vp, _c_i64, _vp, ctypes.c_int, _vp, _vp, _c_i64, _vp, _vp, _vp]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def load(path: str | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library. Raises InternalError if absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise InternalError(
                f"{_LIB_NAME} not built at {p}; run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the Mapper engine has no CPU fallback)")
        lib = ctypes.CDLL(p)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc == BM_OK:
        return
    msg = load().bm_last_error().decode(errors="replace")
    if rc == BM_ERR_DATA:
        raise DataError(f"{what}: {msg}")
    if rc == BM_ERR_NOMEM:
        raise InternalError(f"{what}: out of device memory: {msg}")
    raise InternalError(f"{what}: {msg}")


def ptr(t) -> int:
    """Raw data pointer of a torch tensor or numpy array (0 for None)."""
    if t is None:
        return 0
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def device_count() -> int:
    n = ctypes.c_int(0)
    load().bm_device_count(ctypes.byref(n))
    return int(n.value)
