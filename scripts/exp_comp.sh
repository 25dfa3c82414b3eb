#!/bin/bash
# Timing experiment: components_kernel register budget (CTAs/SM in __launch_bounds__).
mkdir -p gpurun_out
for m in 16 12 8; do
  B200MAP_NVCC_FLAGS="-DBM_COMP_MINB=$m" python -c "
import sys; sys.path.insert(0, '.')
from paper_2011_03209_b200.build import build_library
build_library(force=True)" > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum --clock-control none -k regex:components_kernel --csv --log-file gpurun_out/exp_comp_$m.csv python scripts/probe_build.py cfg3 2 > /dev/null 2>&1
  python scripts/probe_build.py cfg3 4 > gpurun_out/exp_comp_$m.log 2>&1
done
echo done
