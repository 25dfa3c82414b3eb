"""Deterministic parity cases shared by the golden generator and the tests.

Each case regenerates its fp64 inputs from a seed (numpy default_rng is
stable across machines), so the committed fixtures hold only the
reference's OUTPUTS plus a sha256 of the inputs.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np


def sha(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr, dtype=np.float64).tobytes()).hexdigest()


def gmm(n, d, k, box, seed, sigma=1.0):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-box, box, (k, d))
    return c[rng.integers(0, k, n)] + sigma * rng.standard_normal((n, d))


# ---- named configs (BASELINE.json configs[0], configs[1]) --------------------
def cfg1():
    X = gmm(10_000, 3, 5, 10.0, 1)
    params = dict(filters=[{"kind": "column", "column": "x0"}], n=[10], p=[0.3], eps=0.5,
                  min_pts=5, norm="none", mode="precomputed", threshold=20_000)
    return X, params


def cfg2():
    X = gmm(100_000, 64, 10, 5.0, 2)
    params = dict(filters=[{"kind": "l2-norm"}], n=[20], p=[0.25], eps=10.5, min_pts=5,
                  norm="none", mode="precomputed", threshold=20_000)
    return X, params


# ---- randomized instances ------------------------------------------------------
N_INSTANCES = 60


def instance(seed: int):
    """Blobby cloud + random valid parameters covering lens kinds, 1-D/2-D
    covers, normalisations, both strategy modes and small thresholds (mixed
    summation orders)."""
    rng = np.random.default_rng(50_000 + seed)
    n = int(math.exp(rng.uniform(math.log(40), math.log(1500))))
    d = int(rng.integers(1, 41))
    kb = int(rng.integers(1, 6))
    centers = rng.uniform(-6.0, 6.0, (kb, d))
    X = centers[rng.integers(0, kb, n)] + rng.uniform(0.2, 1.5) * rng.standard_normal((n, d))
    kinds = ["l2-norm", "column", "linf-norm"]
    if d >= 2 and rng.random() < 0.3:
        filters = [{"kind": "column", "column": "x0"}, {"kind": str(rng.choice(kinds[::2]))}]
    else:
        k = str(rng.choice(kinds))
        filters = [{"kind": k, "column": "x0"} if k == "column" else {"kind": k}]
    m = len(filters)
    a = X[rng.integers(0, n, 300)]
    b = X[rng.integers(0, n, 300)]
    dd = np.sqrt(((a - b) ** 2).sum(axis=1))
    eps = max(float(np.quantile(dd[dd > 0], rng.uniform(0.03, 0.5))), 1e-6) if (dd > 0).any() else 1.0
    params = dict(
        filters=filters,
        n=[int(v) for v in rng.integers(1, 13, m)],
        p=[float(v) for v in rng.uniform(0.0, 0.7, m)],
        eps=eps,
        min_pts=int(rng.integers(1, 9)),
        norm=str(rng.choice(["none", "minmax", "l2"])),
        mode=str(rng.choice(["precomputed", "on-the-fly"])),
        threshold=int(rng.choice([20_000, 20_000, 64, 200])),
    )
    return X, params


# ---- exact-tie dataset: cdist order and numpy pairwise order disagree -------
def tie_pairs(d: int = 256, want: int = 12, seed: int = 3):
    """Pairs (a, b) whose cdist distance != numpy pairwise distance; the
    dataset places each pair far from the others and sets eps between the two
    values of the first pair so the strategy modes disagree."""
    from scipy.spatial.distance import cdist

    rng = np.random.default_rng(seed)
    pairs = []
    while len(pairs) < want:
        a = rng.standard_normal(d)
        b = rng.standard_normal(d)
        c = float(cdist(a[None], b[None])[0, 0])
        diff = b - a
        q = float(np.sqrt((diff * diff).sum()))
        if c != q:
            pairs.append((a, b, c, q))
    return pairs


def tie_case():
    pairs = tie_pairs()
    eps = min(pairs[0][2], pairs[0][3])
    pts = []
    for i, (a, b, c, q) in enumerate(pairs):
        # rescale the pair so its distance straddles eps exactly like pair 0:
        # keep pair 0 verbatim, shift the others far apart (translation keeps
        # the summation-order disagreement only for pair 0; the others add
        # structure).
        off = np.zeros_like(a)
        off[0] = 1000.0 * i
        pts.append(a + off)
        pts.append(b + off)
    X = np.vstack(pts)
    params = dict(filters=[{"kind": "column", "column": "x1"}], n=[1], p=[0.0], eps=eps,
                  min_pts=2, norm="none", mode="precomputed", threshold=20_000)
    return X, params


# ---- 2-D PCA lens supplied as FilterValues (config 4 shape, reduced) ----------
def pca2d_case():
    X = gmm(20_000, 64, 10, 5.0, 4)
    Xc = X - X.mean(axis=0)
    _, _, vt = np.linalg.svd(Xc[:4000], full_matrices=False)
    F = np.ascontiguousarray(Xc @ vt[:2].T)
    return X, F, dict(n=[15, 15], p=[0.3, 0.3], eps=11.0, min_pts=5)


def pca_fixture_F(X: np.ndarray) -> np.ndarray:
    Xc = X - X.mean(axis=0)
    _, _, vt = np.linalg.svd(Xc[:4000], full_matrices=False)
    return np.ascontiguousarray(Xc @ vt[:2].T)
