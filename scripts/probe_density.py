"""Probe: eps-pairs (distinct, i<j) per cfg3 element vs the pairs the engine
computes in its kept tiles (how much of K3's work lands inside eps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_03209_b200 import engine as eng, workloads  # noqa: E402
from paper_2011_03209_b200 import pipeline as PL  # noqa: E402
from paper_2011_03209_b200.dataset import from_array  # noqa: E402

w = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
X = workloads.points(w)
params = bench.workload_params(w)
dev = torch.device("cuda", 0)
Xd = torch.from_numpy(X).to(dev)
g = PL.build_device(Xd, from_array(X), params, None, None, 0)
st = g.dev_stats
F = g.F
rows, offsets = eng.membership(F, g.cover)
tot_in, tot_all = 0, 0
eps2 = params.eps ** 2
for k in range(len(offsets) - 1):
    r = rows[offsets[k]:offsets[k + 1]]
    P = Xd[r]
    n = len(r)
    cnt = 0
    for a in range(0, n, 4096):
        D = torch.cdist(P[a:a + 4096], P)  # fp64
        cnt += int((D <= params.eps).sum())
    inside = (cnt - n) // 2
    tot_in += inside
    tot_all += n * (n - 1) // 2
    print(f"element {k}: n={n} eps-pairs={inside} frac={inside / max(n * (n - 1) / 2, 1):.4f}", flush=True)
print(f"total eps-pairs {tot_in} of {tot_all} ({tot_in / tot_all:.4f}); engine computed {int(st[0])} "
      f"pairs in kept tiles -> inside fraction of computed {tot_in / int(st[0]):.3f}")
