B200MAP_NVCC_FLAGS="-DBM_COMP_STATS" python -c "
import sys; sys.path.insert(0, '.')
from paper_2011_03209_b200.build import build_library
build_library(force=True)" > gpurun_out/profbuild.log 2>&1
python scripts/probe_build.py cfg3 2 > gpurun_out/compstats.log 2>&1; echo "rc=$?"
