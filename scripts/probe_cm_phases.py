"""Phase timings of compute_mapper at cfg3 (dev tool): device build, result
read-back, graph object assembly, canonical JSON."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2011_03209_b200 import workloads, from_array, compute_mapper
from paper_2011_03209_b200 import pipeline as PL, engine as eng, nerve as NV
from paper_2011_03209_b200.device import require_gpu, to_device_f64

w = workloads.CONFIGS["cfg3"]
X = workloads.points(w)
Xh = torch.from_numpy(X).pin_memory()
pc = from_array(Xh.numpy())
params = bench.workload_params(w)
for _ in range(2):
    compute_mapper(pc, params)
dev = require_gpu()
for rep in range(3):
    T = {}
    sync = lambda: torch.cuda.current_stream(dev).synchronize()
    t = time.perf_counter(); t0 = t
    def mark(k):
        global t
        sync(); n = time.perf_counter(); T[k] = (n - t) * 1e3; t = n
    Xd = to_device_f64(pc.points, dev); mark("h2d")
    Xn = eng.normalize(Xd, params.norm); mark("normalize")
    g = PL.build_device(Xn, pc, params, None, None, 0); mark("build")
    st, fm = eng.node_payload(Xn, g.F, g.node_rows, g.node_off, g.n_nodes); mark("payload")
    host = [PL._pinned_copy(x) for x in (g.F, g.node_rows, g.node_off, st, fm)]; mark("d2h")
    fv_np, rows_np, off_np, st_np, fm_np = (h.numpy() for h in host)
    manifest = params.manifest()
    manifest["intervals"] = [[[iv.lo, iv.hi] for iv in axis] for axis in g.cover.axes]
    graph = NV.assemble_graph(pc, None, g.cover, manifest, rows_np, off_np, g.node_elem, st_np,
                              fm_np, g.edges); mark("assemble")
    b = NV.graph_to_json(graph); mark("json")
    T["total"] = (time.perf_counter() - t0) * 1e3
    print(" ".join(f"{k}={v:.1f}" for k, v in T.items()), len(b))
t = time.perf_counter()
for _ in range(3):
    compute_mapper(pc, params)
print("compute_mapper ms", (time.perf_counter() - t) / 3 * 1e3)
# JSON writer breakdown
import ctypes, numpy as np
f = graph._flat
for _ in range(3):
    t = time.perf_counter(); nb = NV._nodes_json_native(f); t1 = time.perf_counter()
    edges = NV.to_canonical_json([{"s": s, "t": t_, "w": w_} for s, t_, w_ in graph.edges]); t2 = time.perf_counter()
    man = NV.to_canonical_json(graph.manifest); t3 = time.perf_counter()
    out = NV.graph_to_json(graph); t4 = time.perf_counter()
    print(f"nodes_native={1e3*(t1-t):.2f} edges={1e3*(t2-t1):.2f} manifest={1e3*(t3-t2):.2f} graph_to_json={1e3*(t4-t3):.2f}")
