import time, sys
sys.path.insert(0, ".")
import bench, torch
from paper_2011_03209_b200 import workloads, from_array, compute_mapper
from paper_2011_03209_b200 import engine as eng
from paper_2011_03209_b200.pipeline import build_device
from paper_2011_03209_b200.device import require_gpu, to_device_f64
w = workloads.CONFIGS["cfg3"]; X = workloads.points(w); pc = from_array(X); params = bench.workload_params(w)
dev = require_gpu(); Xd = to_device_f64(X, dev)
g = build_device(Xd, pc, params, bench.BUDGET, None, 0)
torch.cuda.synchronize(); print("build ok", g.n_nodes, g.node_rows.shape, g.node_off.shape, g.F.shape, flush=True)
st, fm = eng.node_payload(Xd, g.F, g.node_rows, g.node_off, g.n_nodes)
torch.cuda.synchronize(); print("payload ok", st.shape, fm.shape, flush=True)
for i in range(2):
    t = time.time(); run = compute_mapper(pc, params); print("compute_mapper s", round(time.time() - t, 3), len(run.graph_bytes), flush=True)
