"""Probe: N device-resident builds of a workload (for ncu launch lists / A-B of env knobs).

    python scripts/probe_build.py [cfg3] [steps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import torch  # noqa: E402

from bench import BUDGET, workload_params  # noqa: E402
from paper_2011_03209_b200 import from_array, workloads  # noqa: E402
from paper_2011_03209_b200.device import require_gpu  # noqa: E402
from paper_2011_03209_b200.pipeline import build_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = workloads.CONFIGS[name]
X = workloads.points(w)
dev = require_gpu()
Xd = torch.from_numpy(X).to(dev)
pc = from_array(X)
params = workload_params(w)
for i in range(steps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = build_device(Xd, pc, params, BUDGET, None, 0)
    torch.cuda.synchronize()
    print(f"build {i}: {1e3 * (time.perf_counter() - t):.2f} ms, {g.n_nodes} nodes, "
          f"stats {list(g.dev_stats)}", flush=True)
