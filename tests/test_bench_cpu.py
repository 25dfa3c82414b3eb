"""CPU: the reference-timing helpers behind bench.py's CPU baseline and
`--impl reference` arm (oracle/ref_timing.py, bench.RefSampler): the
whole-build port equals the oracle's graph, the sampling model covers every
element, and the reported time is a lower bound that never exceeds the
pool-schedule simulation."""

import numpy as np

import bench
from oracle import mapper_oracle as O
from oracle import ref_timing as RT
from paper_2011_03209_b200 import workloads


def test_rows_for_budget_monotone():
    sizes = np.array([10, 1000, 50000, 0])
    r1 = bench.rows_for_budget(sizes, 256, 1.0)
    r2 = bench.rows_for_budget(sizes, 256, 100.0)
    assert 1 <= r1 <= r2 <= sizes.max()


def test_schedule_makespan():
    assert RT.schedule_makespan([5, 1, 1, 1], 2) == 5
    assert RT.schedule_makespan([1, 1, 1, 1], 2) == 2
    assert RT.schedule_makespan([], 4) == 0


def test_full_build_port_matches_oracle():
    w = workloads.CONFIGS["cfg1"]
    X = workloads.points(w)
    r = RT.full_build(X, bench.ref_lenses(w), list(w.intervals), list(w.overlaps), w.eps,
                      w.min_pts, workers=2)
    want = O.mapper_graph(X, [("column", 0)], [10], [0.3], w.eps, w.min_pts)
    assert r["nodes"] == len(want["node_rows"]) and r["edges"] == len(want["edges"])
    assert r["seconds"] > 0 and r["single_worker_cluster_s"] > 0


def test_ref_sampler_lower_bound():
    w = workloads.CONFIGS["cfg1"]
    rs = bench.RefSampler(workloads.points(w), w, 2)
    rs.step(0.2, seed=0)
    rs.step(0.2, seed=1)
    rs.critical(0.2)
    est = rs.estimate()
    assert (rs.rows[rs.sizes > 0] > 0).all()  # every element sampled
    assert est["seconds_full_build"] <= est["fifo_contended_s"] * 1.5 + 1.0
    assert est["value"] > 0 and 0 < est["sampled_pair_fraction"] <= 1.0
