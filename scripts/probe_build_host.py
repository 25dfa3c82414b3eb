import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cProfile, pstats
import bench
from paper_2011_03209_b200 import workloads, from_array
from paper_2011_03209_b200.pipeline import build_device
from paper_2011_03209_b200.device import require_gpu, to_device_f64
w = workloads.CONFIGS["cfg3"]; X = workloads.points(w); pc = from_array(X); params = bench.workload_params(w)
dev = require_gpu(); Xd = to_device_f64(X, dev)
for _ in range(3): build_device(Xd, pc, params)
torch.cuda.synchronize()
for _ in range(3):
    g = build_device(Xd, pc, params, sync_timings=True); print({k: round(v*1e3, 2) for k, v in g.timings.items()})
pr = cProfile.Profile(); pr.enable()
for _ in range(5): build_device(Xd, pc, params)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
