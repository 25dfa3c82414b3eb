#!/bin/bash
# GPU iteration: tests, bench, launch list, cfg5 + library-piece probes, a
# functional check of the N-rank bench (ranks share the one GPU over gloo),
# compute_mapper phase timings, then the profiling build (TC MMA-warp waits,
# components path counters).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x ${1:-} > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
tail -3 gpurun_out/pytest.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
python scripts/probe_build.py cfg5 3 > gpurun_out/probe_cfg5.log 2>&1; echo "cfg5 rc=$?"
python scripts/probe_pieces.py > gpurun_out/probe_pieces.log 2>&1; echo "pieces rc=$?"
B200MAP_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 1 --config cfg2 \
  > gpurun_out/bench_n2_gloo.log 2>&1; echo "n2 gloo rc=$?"
B200MAP_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 2 --warmup 1 --impl reference --config cfg1 \
  > gpurun_out/bench_n2_ref.log 2>&1; echo "n2 ref rc=$?"
python scripts/probe_cm_phases.py > gpurun_out/cm_phases.log 2>&1; echo "cm phases rc=$?"
B200MAP_NVCC_FLAGS="-DBM_TC_PROFILE -DBM_COMP_STATS" python -c "
import sys; sys.path.insert(0, '.')
from paper_2011_03209_b200.build import build_library
build_library(force=True)" > gpurun_out/profbuild.log 2>&1
B200MAP_TC_PROFILE=1 python scripts/probe_build.py cfg3 3 > gpurun_out/tcprof.log 2>&1; echo "tcprof rc=$?"
