"""Split the bench's end-to-end step: H2D alone, build alone, both (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2011_03209_b200 import workloads, from_array
from paper_2011_03209_b200.pipeline import build_device
from paper_2011_03209_b200.device import require_gpu
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
w = workloads.CONFIGS["cfg3"]
X = workloads.points(w)
pc = from_array(X)
params = bench.workload_params(w)
dev = require_gpu()
Xh = torch.from_numpy(X).pin_memory()
Xd = Xh.to(dev)
for _ in range(3):
    build_device(Xd, pc, params, bench.BUDGET, None, 0)
torch.cuda.synchronize()
def timeit(fn, n=5):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / n * 1e3
print("h2d ms", timeit(lambda: Xh.to(dev, non_blocking=True)))
buf = torch.empty_like(Xd)
print("h2d copy_ ms", timeit(lambda: buf.copy_(Xh, non_blocking=True)))
print("build ms", timeit(lambda: build_device(Xd, pc, params, bench.BUDGET, None, 0)))
def both():
    Xs = Xh.to(dev, non_blocking=True)
    g = build_device(Xs, pc, params, bench.BUDGET, None, 0)
    g.node_rows.cpu(); g.node_off.cpu()
print("both ms", timeit(both))
def both2():
    buf.copy_(Xh, non_blocking=True)
    g = build_device(buf, pc, params, bench.BUDGET, None, 0)
    g.node_rows.cpu(); g.node_off.cpu()
print("both (reused buffer) ms", timeit(both2))
