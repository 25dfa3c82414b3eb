#!/bin/bash
# Quick GPU iteration: tensor-core/DBSCAN tests, bench, launch list, TC profile.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_tc.py tests/test_gpu_dbscan.py tests/test_gpu_stress.py -q -x > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_q.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
B200MAP_NVCC_FLAGS="-DBM_TC_PROFILE" python -c "
import sys; sys.path.insert(0, '.')
from paper_2011_03209_b200.build import build_library
build_library(force=True)" > gpurun_out/profbuild.log 2>&1
B200MAP_TC_PROFILE=1 python scripts/probe_build.py cfg3 3 > gpurun_out/tcprof.log 2>&1; echo "tcprof rc=$?"
