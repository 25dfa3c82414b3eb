"""Synthetic workloads of BASELINE.json's configs.

Generator (test_acceptance.py:100-104 recipe): rng = default_rng(seed);
C = rng.uniform(-box, box, (K, d)); X = C[rng.integers(0, K, N)] +
sigma * rng.standard_normal((N, d)); fp64, sigma = 1, norm = none.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    d: int
    k: int
    box: float
    seed: int
    lens: tuple          # ((kind, column_or_None), ...) or ("pca2",)
    intervals: tuple
    overlaps: tuple
    eps: float
    min_pts: int = 5
    threshold: int = 10 ** 9  # DistanceStrategy threshold (>= max n_k: every element cdist order)


CONFIGS = {
    "cfg1": Workload("cfg1", 10_000, 3, 5, 10.0, 1, (("column", "x0"),), (10,), (0.3,), 0.5),
    "cfg2": Workload("cfg2", 100_000, 64, 10, 5.0, 2, (("l2-norm", None),), (20,), (0.25,), 10.5),
    "cfg3": Workload("cfg3", 1_000_000, 256, 10, 5.0, 3, (("l2-norm", None),), (40,), (0.3,), 21.3),
    "cfg4": Workload("cfg4", 500_000, 128, 10, 5.0, 4, ("pca2",), (15, 15), (0.3, 0.3), 14.7),
    "cfg5": Workload("cfg5", 4_000_000, 256, 10, 5.0, 5, (("l2-norm", None),), (10,), (0.3,), 21.3),
    # cfg3-shaped at the reference's DEFAULT strategy (threshold 20,000): 5
    # elements of 20-22k rows take numpy's pairwise (on-the-fly) order
    # (tests/golden/cases.py cfg3_default; golden made by nervemap itself)
    "cfg3d": Workload("cfg3d", 200_000, 256, 10, 5.0, 6, (("l2-norm", None),), (40,), (0.3,),
                      21.3, threshold=20_000),
}


def pca2_lens(X: np.ndarray) -> np.ndarray:
    """cfg4's lens: the top-2 principal-component projection (the reference's
    analysis.pca, analysis.py:225-256, is not a FilterSpec kind, so the lens
    is computed on the host and passed as FilterValues to both sides; SVD of
    the centred first 20,000 rows)."""
    Xc = X - X.mean(axis=0)
    _, _, vt = np.linalg.svd(Xc[:20000], full_matrices=False)
    return np.ascontiguousarray(Xc @ vt[:2].T)


def generate(n: int, d: int, k: int, box: float, seed: int, sigma: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-box, box, (k, d))
    return centers[rng.integers(0, k, n)] + sigma * rng.standard_normal((n, d))


def points(w: Workload, n: int | None = None) -> np.ndarray:
    """The workload's fp64 points (optionally only the first n rows)."""
    X = generate(w.n, w.d, w.k, w.box, w.seed)
    return X if n is None else np.ascontiguousarray(X[:n])
