#!/bin/bash
# Timing experiment: K3 with work units of 16 / 32 / 64 column tiles.
mkdir -p gpurun_out
for u in 16 32 64; do
  B200MAP_NVCC_FLAGS="-DBM_TC_UNIT=$u" python -c "
import sys; sys.path.insert(0, '.')
from paper_2011_03209_b200.build import build_library
build_library(force=True)" > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_adjacency --csv --log-file gpurun_out/exp_unit_$u.csv python scripts/probe_build.py cfg3 2 > /dev/null 2>&1
  python scripts/probe_build.py cfg3 4 > gpurun_out/exp_unit_$u.log 2>&1
done
echo done
