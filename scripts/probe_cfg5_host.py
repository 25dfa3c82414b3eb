"""Probe: cfg5 builds with host-side stage marks and torch reserved memory (dev tool)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2011_03209_b200 import workloads, from_array
from paper_2011_03209_b200 import pipeline as PL
w = workloads.CONFIGS["cfg5"]
X = workloads.points(w)
Xd = torch.from_numpy(X).cuda()
pc = from_array(X)
params = bench.workload_params(w)
for i in range(6):
    torch.cuda.synchronize(); t = time.perf_counter()
    g = PL.build_device(Xd, pc, params, None, None, 0, sync_timings=True)
    torch.cuda.synchronize()
    tt = g.timings
    print(f"build {i}: {1e3*(time.perf_counter()-t):.1f} ms  host marks " + " ".join(f"{k}={1e3*v:.1f}" for k, v in tt.items() if k != 'events'), "mem reserved GB", torch.cuda.memory_reserved() / 1e9, flush=True)
