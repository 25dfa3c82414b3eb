#!/bin/bash
# TC kernel profile counters only (profiling build, cfg3 probe).
mkdir -p gpurun_out
B200MAP_NVCC_FLAGS="-DBM_TC_PROFILE" python -c "
import sys; sys.path.insert(0, '.')
from paper_2011_03209_b200.build import build_library
build_library(force=True)" > gpurun_out/profbuild.log 2>&1
B200MAP_TC_PROFILE=1 python scripts/probe_build.py cfg3 3 > gpurun_out/tcprof.log 2>&1; echo "tcprof rc=$?"
