"""eps-pair density of cfg3's largest-element-sized slab vs the pairs the
pruned tile list computes (dev tool: how much work finer pruning could save)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2011_03209_b200 import workloads, engine as eng
from paper_2011_03209_b200.device import require_gpu, to_device_f64
w = workloads.CONFIGS["cfg3"]
X = workloads.points(w)
dev = require_gpu()
Xd = to_device_f64(X, dev)
nrm = np.linalg.norm(X, axis=1)
o = np.argsort(nrm)
n = 133385
mid = len(o) // 2
rows = np.sort(o[mid - n // 2: mid - n // 2 + n])
be = eng.BigElement(Xd, torch.from_numpy(rows).to(dev), w.eps, w.min_pts, 1)
cnt = be.zeros()
be.counts(0, be.tiles, cnt)
torch.cuda.synchronize()
st = be.stats()
c = cnt.cpu().numpy().astype(np.int64)
print("rows", n, "tiles", be.tiles, "eps-pairs (ordered, incl self)", c.sum(),
      "mean nbrs", c.sum() / n, "stats", st.tolist())
print("pairs in computed tiles / eps pairs:", st[0] / max(1, c.sum()))
