"""CPU: the C-ABI library loads, exports every symbol include/b200map.h
declares, and rejects bad arguments with BM_ERR_DATA before touching a GPU."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2011_03209_b200 import _native
from paper_2011_03209_b200.build import build_library

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "b200map.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|const char\*)\s+(bm_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    build_library()
    return _native.load()


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_native.exported_symbols())


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\b(bm_\w+)\b", out))
    for sym in declared_symbols():
        assert sym in exported, sym
        assert getattr(lib, sym) is not None


def test_abi_version_and_error_string(lib):
    assert lib.bm_abi_version() == 1
    assert isinstance(lib.bm_last_error(), bytes)


def test_bad_arguments_are_data_errors(lib):
    # rejected during argument validation: no device work is attempted
    rc = lib.bm_lens_f64(_native.LENS_L2, None, 10, 0, 0, None, None)
    assert rc == _native.BM_ERR_DATA
    assert b"shape" in lib.bm_last_error()
    rc = lib.bm_lens_f64(99, None, 0, 3, 0, None, None)
    assert rc == _native.BM_OK  # n == 0 is a no-op
    rc = lib.bm_normalize_f64(7, None, 4, 2, None, None)
    assert rc == _native.BM_ERR_DATA
    stats = np.zeros(8, dtype=np.int64)
    ncl = np.zeros(1, dtype=np.int32)
    offs = np.array([0, 3], dtype=np.int64)
    order = np.zeros(1, dtype=np.uint8)
    rc = lib.bm_cluster_elements(None, 5, 2, None, offs.ctypes.data, 1, ctypes.c_double(-1.0), 3,
                                 order.ctypes.data, 0, None, ncl.ctypes.data, stats.ctypes.data,
                                 None)
    assert rc == _native.BM_ERR_DATA and b"eps" in lib.bm_last_error()
    rc = lib.bm_cluster_elements(None, 5, 2, None, offs.ctypes.data, 1, ctypes.c_double(1.0), 0,
                                 order.ctypes.data, 0, None, ncl.ctypes.data, stats.ctypes.data,
                                 None)
    assert rc == _native.BM_ERR_DATA and b"min-pts" in lib.bm_last_error()


def test_status_maps_to_exceptions(lib):
    from paper_2011_03209_b200.errors import DataError

    lib.bm_normalize_f64(7, None, 4, 2, None, None)
    with pytest.raises(DataError):
        _native.check(_native.BM_ERR_DATA, "normalize")


def test_no_gpu_means_loud_failure():
    """The product path has no CPU fallback."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2011_03209_b200 import DataError, InternalError, from_array, FilterSpec
    from paper_2011_03209_b200.filters import evaluate

    pc = from_array(np.ones((4, 2)))
    with pytest.raises(InternalError):
        evaluate(pc, FilterSpec(kind="l2-norm"))
    assert not issubclass(InternalError, DataError)


def test_native_graph_json_matches_python_writer():
    """bm_json_nodes (host code, no GPU) writes the node array byte-identically
    to the Python canonical writer, floats included ("%.9g", -0 -> 0)."""
    import numpy as np

    from paper_2011_03209_b200.nerve import assemble_graph, graph_to_json, graph_to_obj
    from paper_2011_03209_b200.nerve import to_canonical_json

    class PC:
        numerical_columns = ["b", "a", "Z", "x_1", "é"]
        categorical_columns = []

    class Cov:
        def __init__(self, two_d):
            self.two_d = two_d

        def element_key(self, k):
            return [k // 3, k % 3] if self.two_d else k

    rng = np.random.default_rng(7)
    specials = [0.0, -0.0, 1e-5, 9.99999999e-5, 1e-4, 123456789.0, 1234567890.0, 1e16,
                -2.5e-300, 5e-324, 1.7976931348623157e308, 0.1, 1 / 3, -7.0, 100.0]
    for two_d in (False, True):
        n_nodes = 40
        sizes = rng.integers(1, 60, n_nodes)
        off = np.zeros(n_nodes + 1, dtype=np.int64)
        np.cumsum(sizes, out=off[1:])
        rows = np.concatenate([np.sort(rng.choice(10 ** 6, s, replace=False)) for s in sizes])
        stats = rng.standard_normal((n_nodes, 5)) * 10.0 ** rng.integers(-12, 12, (n_nodes, 5))
        stats.flat[: len(specials)] = specials
        fmean = rng.standard_normal((n_nodes, 2)) * 1e3
        g = assemble_graph(PC(), None, Cov(two_d), {"k": [1, 2.5], "s": "x"}, rows, off,
                           np.arange(n_nodes), stats, fmean,
                           np.array([[0, 1, 3], [2, 5, 1]], dtype=np.int64))
        assert graph_to_json(g) == to_canonical_json(graph_to_obj(g))


def test_native_graph_json_random_bit_patterns():
    """The native "%.9g" (std::to_chars) equals Python's on random fp64 bit
    patterns: subnormals, huge and tiny exponents, both signs."""
    import numpy as np

    from paper_2011_03209_b200.nerve import assemble_graph, graph_to_json, graph_to_obj
    from paper_2011_03209_b200.nerve import to_canonical_json

    class PC:
        numerical_columns = [f"c{i:02d}" for i in range(64)]
        categorical_columns = []

    class Cov:
        two_d = False

        def element_key(self, k):
            return k

    rng = np.random.default_rng(11)
    n_nodes = 64
    bits = rng.integers(0, 2 ** 63, (n_nodes, 64), dtype=np.int64)
    bits ^= rng.integers(0, 2, (n_nodes, 64), dtype=np.int64) << 63
    stats = bits.view(np.float64).copy()
    stats[~np.isfinite(stats)] = 1.25
    stats[:8] = rng.standard_normal((8, 64)) * 10.0 ** rng.integers(-320, 300, (8, 64))
    off = np.arange(n_nodes + 1, dtype=np.int64) * 3
    rows = np.arange(3 * n_nodes, dtype=np.int64)
    fmean = rng.standard_normal((n_nodes, 1))
    g = assemble_graph(PC(), None, Cov(), {}, rows, off, np.arange(n_nodes), stats, fmean,
                       np.zeros((0, 3), dtype=np.int64))
    assert graph_to_json(g) == to_canonical_json(graph_to_obj(g))
