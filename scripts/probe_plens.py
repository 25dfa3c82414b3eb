"""Time the eccentricity lens at cfg3 size (1M x 256 vs the 50k subsample)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_03209_b200 import workloads, from_array, FilterSpec
from paper_2011_03209_b200.filters import evaluate_device
from paper_2011_03209_b200.device import require_gpu, to_device_f64
w = workloads.CONFIGS["cfg3"]
X = workloads.points(w)
pc = from_array(X)
dev = require_gpu()
Xd = to_device_f64(X, dev)
for spec in (FilterSpec(kind="eccentricity"), FilterSpec(kind="density")):
    for _ in range(2):
        torch.cuda.synchronize(); t = time.time()
        f = evaluate_device(Xd, pc, spec)
        torch.cuda.synchronize(); print(spec.kind, "%.3f s" % (time.time() - t), flush=True)
