"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `nervemap` from /root/reference/pkg/src (read-only; bytecode
writing disabled), runs the cases in cases.py through the reference's own
public API (compute_mapper, or the library pieces for the 2-D PCA lens, as
test_nerve.py:23-30 composes them) and stores the reference's canonical
graph JSON plus a sha256 of each case's inputs. The GPU box never reads
/root/reference: tests compare against these files only.
"""

from __future__ import annotations

import os
import sys
import time

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

import cases  # noqa: E402
from nervemap.clustering import (DbscanParams, DistanceStrategy, cluster_all)  # noqa: E402
from nervemap.cover import build_cover, membership  # noqa: E402
from nervemap.dataset import ColumnSpec, PointCloud  # noqa: E402
from nervemap.errors import DataError  # noqa: E402
from nervemap.filters import FilterSpec, FilterValues  # noqa: E402
from nervemap.nerve import build_graph, graph_to_json  # noqa: E402
from nervemap.pipeline import MapperParams, compute_mapper  # noqa: E402


def cloud(X):
    cols = [ColumnSpec(f"x{j}", "numerical", j) for j in range(X.shape[1])]
    return PointCloud(points=np.ascontiguousarray(X), categorical={}, columns=cols)


def ref_params(p):
    return MapperParams(
        filters=[FilterSpec.from_json_obj(f) for f in p["filters"]], n=p["n"], p=p["p"],
        eps=p["eps"], min_pts=p["min_pts"], norm=p["norm"],
        strategy=DistanceStrategy(mode=p["mode"], threshold=p["threshold"]))


def run(X, p, threads=1):
    try:
        return compute_mapper(cloud(X), ref_params(p), threads=threads).graph_bytes
    except DataError as e:
        return ("DataError: " + str(e)).encode()


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def as_u8(b: bytes):
    return np.frombuffer(b, dtype=np.uint8)


def near_eps():
    """Planted near-eps links in 256-D (cases.near_eps_case), both modes."""
    X, p = cases.near_eps_case()
    pre = run(X, dict(p, mode="precomputed"))
    fly = run(X, dict(p, mode="on-the-fly"))
    assert pre != fly, "near-eps case does not separate the strategy modes"
    save("near_eps", x_sha=np.array(cases.sha(X)), **compact("pre", pre), **compact("fly", fly))


def compact(prefix, graph_bytes):
    """A large graph JSON as its sha256 plus node rows and edges (the JSON
    carries 256 column means per node; the hash pins every byte of it)."""
    import hashlib
    import json

    g = json.loads(graph_bytes)
    rows = [nd["rows"] for nd in g["nodes"]]
    return {f"{prefix}_sha": np.array(hashlib.sha256(graph_bytes).hexdigest()),
            f"{prefix}_node_off": np.cumsum([0] + [len(r) for r in rows]).astype(np.int64),
            f"{prefix}_node_rows": (np.concatenate([np.asarray(r, dtype=np.int32) for r in rows])
                                    if rows else np.zeros(0, np.int32)),
            f"{prefix}_edges": np.array([(e["s"], e["t"], e["w"]) for e in g["edges"]],
                                        dtype=np.int64).reshape(-1, 3)}


def main():
    if len(sys.argv) > 1:  # named pieces only, e.g. `make_golden.py near_eps`
        for name in sys.argv[1:]:
            t = time.time()
            globals()[name]()
            print(name, time.time() - t)
        return
    threads = os.cpu_count() or 1
    t = time.time()
    X, p = cases.cfg1()
    save("cfg1", graph=as_u8(run(X, p, threads)), x_sha=np.array(cases.sha(X)))
    print("cfg1", time.time() - t)

    t = time.time()
    X, p = cases.cfg2()
    save("cfg2", graph=as_u8(run(X, p, threads)), x_sha=np.array(cases.sha(X)))
    print("cfg2", time.time() - t)

    t = time.time()
    graphs, shas = {}, []
    for s in range(cases.N_INSTANCES):
        X, p = cases.instance(s)
        graphs[f"g{s}"] = as_u8(run(X, p))
        shas.append(cases.sha(X))
    save("instances", x_sha=np.array(shas), **graphs)
    print("instances", time.time() - t)

    X, p = cases.tie_case()
    pre = run(X, dict(p, mode="precomputed"))
    fly = run(X, dict(p, mode="on-the-fly"))
    assert pre != fly, "tie case does not separate the strategy modes"
    save("tie", pre=as_u8(pre), fly=as_u8(fly), x_sha=np.array(cases.sha(X)))

    X, F, q = cases.pca2d_case()
    pc = cloud(X)
    fv = FilterValues(values=F.copy(), specs=[FilterSpec(kind="l2-norm")] * 2)
    cover = build_cover(fv, q["n"], q["p"])
    members = membership(fv, cover)
    cl = cluster_all(pc, members, DbscanParams(q["eps"], q["min_pts"]), DistanceStrategy(),
                     threads=threads)
    g = build_graph(cl, pc, fv, cover, manifest={"test": True})
    save("pca2d", graph=as_u8(graph_to_json(g)), F=F, x_sha=np.array(cases.sha(X)),
         sizes=np.array([m.size for m in members]))
    near_eps()


if __name__ == "__main__":
    main()
