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


# ---- cfg3-shaped case at the reference's DEFAULT strategy ----------------------
def cfg3_default():
    """200k x 256 Gaussian mixture, l2-norm lens, 40 intervals, 30% overlap,
    eps 21.3, min_pts 5 and the reference's default strategy (precomputed,
    threshold 20,000, 8 GiB budget): 5 elements exceed 20,000 rows and take the
    numpy-pairwise (on-the-fly) order (clustering.py:137-139, 201-208), the
    other 35 the cdist order — both orders at cfg3's dimension and density."""
    X = gmm(200_000, 256, 10, 5.0, 6)
    params = dict(filters=[{"kind": "l2-norm"}], n=[40], p=[0.3], eps=21.3, min_pts=5,
                  norm="none", mode="precomputed", threshold=20_000)
    return X, params


# ---- planted near-eps stress case (256-D, thousands of pairs at +-2 ulp) --------
def _nudge_to(a, b, eps, cd, max_iter=200):
    """Move b by single-ulp steps of its largest-difference coordinates until
    the cdist distance |a - b| lies within 2 ulps of eps (deterministic)."""
    ulp = np.spacing(eps)
    order = np.argsort(-np.abs(b - a), kind="stable")
    for it in range(max_iter):
        dd = cd(a, b)
        if abs(dd - eps) <= 2 * ulp:
            return b, True
        t = order[it % 16]
        step = np.nextafter(b[t], np.inf if (b[t] > a[t]) == (dd < eps) else -np.inf)
        b = b.copy()
        b[t] = step
    return b, False


def near_eps_case(n_pairs: int = 2400, d: int = 256, eps: float = 3.0, seed: int = 77):
    """One cover element (column lens, 1 interval) of `n_pairs` planted links
    whose cdist length is within +-2 ulp of eps; every third link is extended
    to a chain a-b-c (both links planted). Anchors are ~68 apart, so cross
    distances are far from eps and most tile pairs are pruned while the
    planted ones are not. min_pts = 2: each link's eps decision alone decides
    whether its points form a cluster, in both summation orders (which
    disagree on some links)."""
    from scipy.spatial.distance import cdist

    def cd(u, v):
        return float(cdist(u[None], v[None])[0, 0])

    rng = np.random.default_rng(seed)
    pts = []
    for m in range(n_pairs):
        a = 3.0 * rng.standard_normal(d)
        chain = [a]
        for _ in range(2 if m % 3 == 0 else 1):
            u = rng.standard_normal(d)
            u /= np.sqrt((u * u).sum())
            b = chain[-1] + eps * u
            b, _ = _nudge_to(chain[-1], b, eps, cd)
            chain.append(b)
        pts.extend(chain)
    X = np.vstack(pts)
    X = X[rng.permutation(len(X))]  # links spread across tiles and entry order
    params = dict(filters=[{"kind": "column", "column": "x1"}], n=[1], p=[0.0], eps=eps,
                  min_pts=2, norm="none", mode="precomputed", threshold=20_000)
    return X, params
