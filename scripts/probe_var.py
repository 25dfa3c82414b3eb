"""Per-build wall times of 20 consecutive cfg3 builds (dev tool: variance)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2011_03209_b200 import workloads, from_array
from paper_2011_03209_b200.pipeline import build_device
from paper_2011_03209_b200.device import require_gpu, to_device_f64
w = workloads.CONFIGS["cfg3"]
X = workloads.points(w)
pc = from_array(X)
params = bench.workload_params(w)
dev = require_gpu()
Xd = to_device_f64(X, dev)
ts = []
for i in range(23):
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = build_device(Xd, pc, params, bench.BUDGET, None, 0)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t) * 1e3)
print(" ".join(f"{t:.1f}" for t in ts))
sampler = bench.ClockSampler(0)
with sampler:
    ts = []
    for i in range(20):
        torch.cuda.synchronize()
        t = time.perf_counter()
        g = build_device(Xd, pc, params, bench.BUDGET, None, 0)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
print("with nvidia-smi sampler:", " ".join(f"{t:.1f}" for t in ts))
print(os.cpu_count(), "cpus; load", os.getloadavg())
