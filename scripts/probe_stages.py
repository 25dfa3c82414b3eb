"""Fine-grained host/device timing of one cfg3 build (dev tool)."""
import os, sys, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2011_03209_b200 import workloads, FilterSpec, MapperParams, DistanceStrategy, from_array
from paper_2011_03209_b200.pipeline import build_device
from paper_2011_03209_b200.device import require_gpu, to_device_f64

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
w = workloads.CONFIGS[name]
X = workloads.points(w)
pc = from_array(X)
params = MapperParams(filters=[FilterSpec(kind="l2-norm")], n=list(w.intervals), p=list(w.overlaps),
                      eps=w.eps, min_pts=w.min_pts, strategy=DistanceStrategy(threshold=10**9))
dev = require_gpu()
Xd = to_device_f64(X, dev)
for _ in range(3):
    build_device(Xd, pc, params, 1 << 62, None, 0)
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
for _ in range(5):
    build_device(Xd, pc, params, 1 << 62, None, 0)
torch.cuda.synchronize()
pr.disable()
print("ms/build", (time.perf_counter() - t) / 5 * 1e3)
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
