"""Quick device timing of the hot path on the named configs (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2011_03209_b200 import workloads, FilterSpec, MapperParams, DistanceStrategy, from_array
from paper_2011_03209_b200.pipeline import build_device
from paper_2011_03209_b200.device import require_gpu, to_device_f64

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg2"]
engine = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dev = require_gpu()
for name in names:
    w = workloads.CONFIGS[name]
    t = time.time(); X = workloads.points(w); tg = time.time() - t
    pc = from_array(X)
    filters = [FilterSpec(kind=k, column=c) if k == "column" else FilterSpec(kind=k) for k, c in w.lens]
    thr = 10**9 if name in ("cfg3", "cfg4", "cfg5") else 20_000
    params = MapperParams(filters=filters, n=list(w.intervals), p=list(w.overlaps), eps=w.eps,
                          min_pts=w.min_pts, strategy=DistanceStrategy(threshold=thr))
    Xd = to_device_f64(X, dev); torch.cuda.synchronize()
    for it in range(2):
        t = time.time()
        g = build_device(Xd, pc, params, budget_bytes=1 << 62, engine=engine, sync_timings=True)
        torch.cuda.synchronize(); el = time.time() - t
        print(f"{name} it{it} engine={engine} total={el:.3f}s stages={ {k: round(v,4) for k,v in g.timings.items()} } "
              f"nodes={g.n_nodes} edges={len(g.edges)} sum_nk={int(g.sizes.sum())} max_nk={int(g.sizes.max())} "
              f"sum_nk2={float((g.sizes.astype(np.float64)**2).sum()):.3e} adj_ms={g.dev_stats[5]/1e6:.1f} pre_ms={g.dev_stats[6]/1e6:.1f} post_ms={g.dev_stats[7]/1e6:.1f} rechecks={g.dev_stats[1]} kept={1-g.dev_stats[2]/max(g.dev_stats[3],1):.3f} gen={tg:.1f}s", flush=True)
