#!/bin/bash
# The GPU test suite on the debug build (-DBM_DEBUG_BOUNDS: device-side bounds
# assertions in the tensor-core, recheck, quantiser, projection and
# union-find kernels trap on a bad index). compute-sanitizer is closed on
# this GPU pool, so this is the memory-safety check we can run.
mkdir -p gpurun_out
B200MAP_NVCC_FLAGS="-DBM_DEBUG_BOUNDS" python -c "
import sys; sys.path.insert(0, '.')
from paper_2011_03209_b200.build import build_library
build_library(force=True, verbose=True)" > gpurun_out/debug_build.log 2>&1
grep -c BM_DASSERT paper_2011_03209_b200/csrc/*.cu* >> gpurun_out/debug_build.log
cuobjdump -sass paper_2011_03209_b200/libb200map.so | grep -c "BPT.TRAP\|TRAP" >> gpurun_out/debug_build.log
python -m pytest tests -m gpu -q > gpurun_out/debug_pytest.log 2>&1; echo "debug pytest rc=$?" | tee -a gpurun_out/debug_pytest.log
python scripts/probe_build.py cfg3 2 > gpurun_out/debug_cfg3.log 2>&1; echo "debug cfg3 rc=$?" | tee -a gpurun_out/debug_cfg3.log
