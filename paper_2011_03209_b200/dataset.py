"""Point-cloud data model (mirrors nervemap/dataset.py:25-97, 165-186).

The Mapper engine only needs the read-only fp64 coordinate matrix and column
metadata; CSV wrangling stays with the caller (nervemap.dataset.wrangle, out
of scope here). Any object with the same attributes (e.g. a nervemap
PointCloud) is accepted by the engine.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DataError

NORMALIZATIONS = ("none", "minmax", "l2")


@dataclass(frozen=True)
class ColumnSpec:
    name: str
    kind: str  # "numerical" | "categorical"
    index: int


@dataclass(frozen=True)
class PointCloud:
    """Dataset X: points[i] = row i over the numerical columns (header order)."""

    points: np.ndarray
    categorical: dict
    columns: list
    metric: str = "euclidean"

    def __post_init__(self):
        self.points.setflags(write=False)

    @property
    def n_rows(self) -> int:
        return self.points.shape[0]

    @property
    def n_dims(self) -> int:
        return self.points.shape[1]

    @property
    def numerical_columns(self) -> list[str]:
        return [c.name for c in self.columns if c.kind == "numerical"]

    @property
    def categorical_columns(self) -> list[str]:
        return [c.name for c in self.columns if c.kind == "categorical"]

    def numerical_index(self, name: str) -> int:
        pos = 0
        for c in self.columns:
            if c.kind != "numerical":
                continue
            if c.name == name:
                return pos
            pos += 1
        if any(c.name == name for c in self.columns):
            raise DataError(f"column {name!r} is categorical")
        raise DataError(f"unknown column {name!r}")

    def column_values(self, name: str) -> np.ndarray:
        return self.points[:, self.numerical_index(name)]


def from_array(points, names=None) -> PointCloud:
    """PointCloud straight from an (N, d) numeric matrix (no wrangling)."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    pts = np.ascontiguousarray(pts)
    names = names or [f"x{j}" for j in range(pts.shape[1])]
    cols = [ColumnSpec(nm, "numerical", j) for j, nm in enumerate(names)]
    return PointCloud(points=pts, categorical={}, columns=cols)


def normalize(pc: PointCloud, scheme: str) -> PointCloud:
    """Rescaled copy computed on the GPU (bit-identical to dataset.py:176-185)."""
    if scheme not in NORMALIZATIONS:
        raise DataError(f"unknown normalization {scheme!r}")
    if scheme == "none":
        return pc
    from . import engine
    from .device import require_gpu, to_device_f64

    dev = require_gpu()
    out = engine.normalize(to_device_f64(pc.points, dev), scheme).cpu().numpy()
    return PointCloud(points=out, categorical=pc.categorical, columns=pc.columns)
