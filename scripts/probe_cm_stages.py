"""Where compute_mapper's end-to-end time goes at cfg3 (dev tool)."""
import os, sys, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2011_03209_b200 import workloads, from_array, compute_mapper
w = workloads.CONFIGS["cfg3"]
X = workloads.points(w)
Xh = torch.from_numpy(X).pin_memory()
pc = from_array(Xh.numpy())
params = bench.workload_params(w)
for _ in range(2):
    compute_mapper(pc, params)
pr = cProfile.Profile()
pr.enable()
t = time.perf_counter()
for _ in range(3):
    compute_mapper(pc, params)
dt = (time.perf_counter() - t) / 3
pr.disable()
print("ms per compute_mapper", dt * 1e3)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
