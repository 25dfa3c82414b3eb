#!/bin/bash
# Evidence run: compute-sanitizer (memcheck, racecheck, synccheck) on small
# builds, ncu --set full of the HBM-bound subsystems and of the dominant kernel.
#   gpurun -- 'bash scripts/evidence.sh [tag]'
mkdir -p gpurun_out
tag=${1:-r02}
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/probe_sanitize.py > gpurun_out/${tag}_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
done
ncu --set full --clock-control none --import-source on \
  -k regex:"membership_kernel|node_keys|radix|entry_pairs|run_pairs|point_slots|point_pairs|dense_edges|lens_l2|node_stats|group" \
  --launch-skip 40 -c 14 -o gpurun_out/${tag}_subsys python scripts/probe_build.py cfg3 3 > gpurun_out/${tag}_ncu_subsys.log 2>&1
echo "ncu subsys rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"tc_adjacency|components_kernel|colcount|recheck|quantize|tile_stats|tile_project|tile_prune" \
  --launch-skip 8 -c 8 -o gpurun_out/${tag}_main python scripts/probe_build.py cfg3 3 > gpurun_out/${tag}_ncu_main.log 2>&1
echo "ncu main rc=$?"
