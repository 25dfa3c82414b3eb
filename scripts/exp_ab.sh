#!/bin/bash
# A/B timing of compile-time variants: bash scripts/exp_ab.sh <kernel-regex> "<flagsA>" "<flagsB>" ...
# (flags "-" = default build). Each variant: cfg3 probe timing + launch list of the kernels.
# PROBE overrides the profiled command (default: scripts/probe_build.py cfg3 2).
mkdir -p gpurun_out
re=$1; shift
i=0
for fl in "$@"; do
  [ "$fl" = "-" ] && fl=""
  B200MAP_NVCC_FLAGS="$fl" python -c "
import sys; sys.path.insert(0, '.')
from paper_2011_03209_b200.build import build_library
build_library(force=True)" > /dev/null 2>&1 || { echo "build $fl failed"; continue; }
  python scripts/probe_build.py cfg3 5 > gpurun_out/ab_$i.log 2>&1
  ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum --clock-control none -k regex:"$re" --csv --log-file gpurun_out/ab_$i.csv ${PROBE:-python scripts/probe_build.py cfg3 2} > /dev/null 2>&1
  echo "== variant $i: '$fl'  $(tail -1 gpurun_out/ab_$i.log | cut -c1-30)"
  python - <<PY
import csv, collections
rows=[r for r in csv.DictReader(l for l in open("gpurun_out/ab_$i.csv") if not l.startswith("=="))]
d=collections.defaultdict(list)
for r in rows: d[(r["Kernel Name"][:40], r["Metric Name"][:12])].append(float(r["Metric Value"].replace(",","")))
for k,v in sorted(d.items()): print("  ", k, [round(x) for x in v])
PY
  i=$((i+1))
done
python -c "
import sys; sys.path.insert(0, '.')
from paper_2011_03209_b200.build import build_library
build_library(force=True)" > /dev/null 2>&1
