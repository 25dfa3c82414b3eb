#!/bin/bash
# e2e checks: cfg3 bench (pinned + pageable), cfg5 bench, cfg4 library-piece phases.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_cfg3.json 2> gpurun_out/e2e_cfg3.err; echo "cfg3 rc=$?"
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_cfg5.json 2> gpurun_out/e2e_cfg5.err; echo "cfg5 rc=$?"
timeout 600 python scripts/probe_pieces.py > gpurun_out/e2e_pieces.log 2>&1; echo "pieces rc=$?"
