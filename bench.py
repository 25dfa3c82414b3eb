"""Benchmark of the Mapper-graph build (BASELINE.json metric) on B200.

A step = one full Mapper graph build of the workload: lens -> cover binning
-> per-element DBSCAN -> nodes -> nerve edges.
  value : points/s with X already resident in HBM (device-timed, CUDA events,
          max over ranks)
  e2e   : points/s through the reference-facing call with HOST buffers: on
          one GPU compute_mapper(pc, params) on page-locked fp64 X, returning
          the MapperRun with the canonical graph JSON (H2D of X, D2H of the
          node rows/payload/edges, JSON writing all inside the timed region);
          on N GPUs the sharded build with X copied H2D and node rows + edges
          copied D2H every step
Inputs (2 GB at 1M x 256 fp64) exceed the 126 MB L2, so no flush is needed.

  python bench.py [--gpus N --steps K --warmup W --config cfg3 --impl ours|reference]
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N (NCCL; elements
sharded by LPT, labels all-gathered to rank 0).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "mapper_graph_build_points_per_s"
UNIT = "points/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--engine", type=int, default=0, help="0 auto, 1 exact fp64, 2 tensor core")
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="target CPU time of the bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def workload_params(w):
    from paper_2011_03209_b200 import DistanceStrategy, FilterSpec, MapperParams

    filters = [FilterSpec(kind=k, column=c) if k == "column" else FilterSpec(kind=k)
               for k, c in w.lens]
    # the 1M-row configs are run with matrices for every
    # element on both sides (threshold >= max n_k), i.e. the cdist order.
    return MapperParams(filters=filters, n=list(w.intervals), p=list(w.overlaps), eps=w.eps,
                        min_pts=w.min_pts, strategy=DistanceStrategy(threshold=10 ** 9))


BUDGET = 1 << 62


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def alg_flops(sizes, d):
    s = np.asarray(sizes, dtype=np.float64)
    return float((2.0 * d * s * (s - 1) / 2.0).sum())


def ncu_traffic(kernel="tc_adjacency_kernel"):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/r01_ncu_full_cfg3.txt)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_full_cfg3.txt")) as f:
            block = None
            for line in f:
                if line.startswith("void ") or line.startswith("unnamed"):
                    block = line
                if block and kernel in block and "dram traffic" in line:
                    return float(line.split()[-1])
    except OSError:
        pass
    return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


# ---------------------------------------------------------------------------
# CPU baseline: the oracle restatement of the reference (fork pool over
# elements, like clustering.py:281-315) on a bounded sample of elements,
# extrapolated to the whole workload by pair work (sum n_k^2 d).
# ---------------------------------------------------------------------------
def cpu_baseline(X, w, sizes, members_fn, target_s, workers):
    from oracle import mapper_oracle as O

    order = np.argsort(sizes)
    # pick small elements until their estimated CPU time reaches the target
    est_rate = 1.2e6 * workers  # n_k^2 per second (measured ~1.3e6 per process on the box)
    chosen, acc = [], 0.0
    for k in order:
        if sizes[k] == 0:
            continue
        chosen.append(int(k))
        acc += float(sizes[k]) ** 2
        if acc / est_rate >= target_s:
            break
    members = members_fn()
    t0 = time.perf_counter()
    O.cluster_all(X, [members[k] for k in chosen], w.eps, w.min_pts,
                  [O.ORDER_SEQUENTIAL] * len(chosen), workers=workers)
    dt = time.perf_counter() - t0
    work_sample = float(sum(float(sizes[k]) ** 2 for k in chosen))
    work_all = float((np.asarray(sizes, dtype=np.float64) ** 2).sum())
    t_full = dt * work_all / max(work_sample, 1.0)
    return {
        "value": w.n / t_full,
        "unit": UNIT,
        "cores": workers,
        "kind": "port",
        "sample": (f"oracle (numpy/scipy restatement of nervemap) DBSCAN of {len(chosen)} of "
                   f"{int((np.asarray(sizes) > 0).sum())} cover elements of {w.name} "
                   f"({100 * work_sample / work_all:.2f}% of the n_k^2 pair work) in {dt:.1f}s on "
                   f"{workers} processes, extrapolated by pair work to {t_full:.0f}s for the "
                   f"whole build (lens/cover/nerve excluded: <1% of reference time)"),
        "seconds_full_estimate": t_full,
    }


def host_members(X, w):
    from oracle import mapper_oracle as O

    F = np.column_stack([O.lens(X, k, int(c[1:]) if c else 0) for k, c in w.lens])
    axes = [O.cover_axis(F[:, a], w.intervals[a], w.overlaps[a]) for a in range(F.shape[1])]
    return O.membership(F, axes)


def run_reference(args, w, rank, world):
    if rank != 0:
        return
    X = __import__("paper_2011_03209_b200.workloads", fromlist=["points"]).points(w)
    members = host_members(X, w)
    sizes = np.array([m.size for m in members])
    workers = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        per_step = max(3.0, args.cpu_seconds / max(args.steps, 1))
        cb = cpu_baseline(X, w, sizes, lambda: members, per_step, workers)
        if i >= args.warmup:
            vals.append(cb)
    v = float(np.median([c["value"] for c in vals]))
    cb = dict(vals[-1])
    cb["value"] = v
    cb.pop("seconds_full_estimate", None)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * w.n / v,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_of(w, world),
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_of(w, world):
    return {"workload": f"{w.name}: {w.n}x{w.d} Gaussian mixture (K={w.k}, box={w.box}, "
                        f"seed={w.seed}), lens={list(w.lens)}, intervals={list(w.intervals)}, "
                        f"overlap={list(w.overlaps)}, eps={w.eps}, min_pts={w.min_pts}",
            "points": w.n, "dims": w.d, "strategy": "precomputed, threshold>=max n_k (cdist order)",
            "parallelism": f"cover elements sharded over {world} GPU(s)",
            "l2": "inputs (N*d*8 bytes) exceed the 126 MB L2; no flush needed"}


def main():
    args = parse()
    from paper_2011_03209_b200 import workloads

    w = workloads.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, w, rank, world)
        return

    import torch

    # B200MAP_DIST_BACKEND=gloo runs the N-rank code path on fewer GPUs (ranks
    # share devices; functional check only — every timing uses NCCL, 1 GPU/rank)
    backend = os.environ.get("B200MAP_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local %= max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    os.environ.setdefault("B200MAP_DEVICE", str(local))
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2011_03209_b200 import _native, engine as eng
    from paper_2011_03209_b200.device import require_gpu
    from paper_2011_03209_b200.distributed import build_distributed
    from paper_2011_03209_b200.pipeline import build_device

    dev = require_gpu()
    lib = _native.load()
    X = workloads.points(w)
    pc = __import__("paper_2011_03209_b200", fromlist=["from_array"]).from_array(X)
    params = workload_params(w)
    Xh = torch.from_numpy(X).pin_memory()
    Xd = Xh.to(dev)
    stream = torch.cuda.current_stream(dev)

    def step(Xdev):
        if world > 1:
            g, st = build_distributed(Xdev, pc, params, rank, world, dist, BUDGET, args.engine)
        else:
            g = build_device(Xdev, pc, params, BUDGET, None, args.engine)
            st = g.dev_stats
        return g, st

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def sum_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up
    for _ in range(args.warmup):
        g, st = step(Xd)
    barrier()

    # ---- device-resident timed region (value)
    adj_ns, pairs_eval, tiles_tot, tiles_skip, sizes = 0, 0, 0, 0, None
    launches0 = lib.bm_launch_count()
    with ClockSampler(local) as clk:
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            g, st = step(Xd)
            adj_ns += int(st[5])
            pairs_eval += int(st[0])
            tiles_tot += int(st[3])
            tiles_skip += int(st[2])
        e1.record(stream)
        barrier()
    launches = lib.bm_launch_count() - launches0
    t_dev = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    adj_s = max_over_ranks(adj_ns / 1e9) / args.steps
    if g is not None:
        sizes = g.sizes

    # ---- end-to-end timed region: host X in (page-locked), result out.
    # One GPU: the reference-facing call itself, compute_mapper(pc, params)
    # (pipeline.py:81-110) -> MapperRun with the canonical graph JSON bytes.
    # Several GPUs: the sharded build + read-back of node rows and edges.
    h2d = X.nbytes
    d2h = 0
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    if world == 1:
        from paper_2011_03209_b200 import compute_mapper, from_array

        pc_host = from_array(Xh.numpy())  # page-locked host buffer, no copy
        run = compute_mapper(pc_host, params, engine=args.engine)
        barrier()
        f0.record(stream)
        for _ in range(args.steps):
            run = compute_mapper(pc_host, params, engine=args.engine)
        f1.record(stream)
        barrier()
        gr = run.graph
        n_rows = sum(len(nd.rows) for nd in gr.nodes)
        d2h = 8 * (n_rows + gr.n_nodes + 1 + gr.n_nodes * (w.d + len(params.filters)) +
                   3 * len(gr.edges))
        e2e_api = "compute_mapper -> MapperRun (graph + canonical JSON bytes)"
    else:
        Xs = torch.empty_like(Xd)  # the step's input buffer (refilled from host every step)
        barrier()
        f0.record(stream)
        for _ in range(args.steps):
            Xs.copy_(Xh, non_blocking=True)
            g2, _ = step(Xs)
            if g2 is not None:
                nr = g2.node_rows.cpu()
                no = g2.node_off.cpu()
                d2h = nr.numel() * 8 + no.numel() * 8 + g2.edges.nbytes
        f1.record(stream)
        barrier()
        e2e_api = "build_distributed -> node rows + edges on rank 0"
    t_e2e = max_over_ranks(f0.elapsed_time(f1) / 1e3)
    # collectives every rank joins before rank 0 alone reports
    pairs_all = sum_over_ranks(pairs_eval)
    tiles_tot = sum_over_ranks(tiles_tot)
    tiles_skip = sum_over_ranks(tiles_skip)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    p, src = peaks()
    F = alg_flops(sizes, w.d)
    # the distance stage computes only the tile pairs the centroid/radius bound
    # cannot exclude: its algorithmic work is one d-dim dot product (2d flop)
    # per distinct row pair inside those tiles (pairs_eval, from the engine)
    F_exec = 2.0 * w.d * pairs_all / args.steps  # all ranks' executed pair work per step
    # per GPU: the ranks' work over the slowest rank's distance-stage time
    achieved = F_exec / world / adj_s / 1e12 if adj_s > 0 else 0.0
    peak = p.get("bf16_tflops_sustained", 1384.6)
    value = w.n * args.steps / t_dev
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64 (exact decisions); distance candidates on tensor cores" if args.engine != 1
        else "f64",
        "data": "synthetic", "config": config_of(w, world),
        "e2e": {"value": w.n * args.steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * t_e2e / args.steps,
                "api": e2e_api},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(),
                     "traffic_note": "DRAM bytes per tc_adjacency_kernel launch, ncu --set full "
                                     "(profiles/r01_ncu_full_cfg3.txt)",
                     "kernel": "eps-adjacency (distance tiles) stage",
                     "kernel_ms_per_step": adj_s * 1e3,
                     "kernel_share_of_step": adj_s / (t_dev / args.steps),
                     "alg_flops_per_step": F_exec, "alg_flops_unpruned_per_step": F,
                     "tile_pairs_pruned_frac": tiles_skip / max(tiles_tot, 1),
                     # exactness costs 6 int8 limb products per credited pair: at
                     # the nominal dense int8 rate (4.5 POPS, B200_PROFILING.md) the
                     # formulation tops out at 750 credited TFLOP/s
                     "ceiling_frac_exact_int8": (4500.0 / 6.0) / peak,
                     "peak_source": f"{src} bf16 sustained"},
        "gpu_launches": int(launches),
        "nodes": int(g.n_nodes), "edges": int(len(g.edges)),
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1:
        members = None

        def members_fn():
            return host_members(X, w)

        line["cpu_baseline"] = {k: v for k, v in cpu_baseline(
            X, w, np.asarray(sizes), members_fn, args.cpu_seconds, os.cpu_count() or 1).items()
            if k != "seconds_full_estimate"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
