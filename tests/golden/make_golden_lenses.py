"""Golden vectors for the O(N x M) lenses (filters.py:103-150), produced by
running the reference itself (nervemap.filters.evaluate) in the build
container: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_lenses.py

Two clouds: 900 points (targets = all points) and 52,000 points (targets =
the reference's seed-1729 subsample of 50,000 rows; default bandwidth from
its 1000-point subsample)."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import cases  # noqa: E402

from nervemap.dataset import PointCloud  # noqa: E402
from nervemap.filters import FilterSpec, evaluate  # noqa: E402

SPECS = {
    "ecc1": dict(kind="eccentricity"),
    "ecc2": dict(kind="eccentricity", p=2.0),
    "ecc3": dict(kind="eccentricity", p=3.0),
    "eccinf": dict(kind="eccentricity", p=float("inf")),
    "dens": dict(kind="density"),
    "dens17": dict(kind="density", bandwidth=1.7),
}


def cloud(X):
    from nervemap.dataset import ColumnSpec

    cols = [ColumnSpec(f"x{j}", "numerical", j) for j in range(X.shape[1])]
    return PointCloud(points=X, categorical={}, columns=cols)


def main():
    out = {}
    for tag, (n, d, seed, names) in {
        "small": (900, 5, 11, list(SPECS)),
        "big": (52_000, 3, 12, ["ecc1", "eccinf", "dens"]),
    }.items():
        X = cases.gmm(n, d, 4, 3.0, seed)
        pc = cloud(X)
        out[f"{tag}_sha"] = np.array(cases.sha(X))
        for name in names:
            out[f"{tag}_{name}"] = evaluate(pc, FilterSpec(**SPECS[name]))
            print(tag, name, flush=True)
    path = os.path.join(HERE, "plens.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path))


if __name__ == "__main__":
    main()
