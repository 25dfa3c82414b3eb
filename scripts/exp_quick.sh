#!/bin/bash
# Rebuild, parity subset (DBSCAN, tensor-core, full-size goldens), cfg3 build
# timing and a launch list of the named kernels.   bash scripts/exp_quick.sh <kernel-regex> [tag]
mkdir -p gpurun_out
re=${1:-components_kernel}; tag=${2:-q}
python -c "
import sys; sys.path.insert(0, '.')
from paper_2011_03209_b200.build import build_library
build_library(force=True)" > gpurun_out/${tag}_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/${tag}_build.log; exit 1; }
python -m pytest tests/test_gpu_dbscan.py tests/test_gpu_tc.py tests/test_gpu_fullsize.py tests/test_gpu_stress.py -q -x > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${tag}_pytest.log
python scripts/probe_build.py cfg3 5 > gpurun_out/${tag}_probe.log 2>&1; tail -2 gpurun_out/${tag}_probe.log | cut -c1-40
ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum --clock-control none -k regex:"$re" --csv --log-file gpurun_out/${tag}_ncu.csv python scripts/probe_build.py cfg3 2 > /dev/null 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.DictReader(l for l in open("gpurun_out/${tag}_ncu.csv") if not l.startswith("=="))]
d=collections.defaultdict(list)
for r in rows: d[(r["Kernel Name"][:40], r["Metric Name"])].append(float(r["Metric Value"].replace(",","")))
for k,v in sorted(d.items()): print(k, len(v), [round(x) for x in v])
PY
