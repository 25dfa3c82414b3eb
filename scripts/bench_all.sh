#!/bin/bash
# Bench lines of every BASELINE config (both arms) into gpurun_out/ (copied to profiles/ by hand).
#   gpurun -- 'bash scripts/bench_all.sh [tag]'
tag=${1:-r02}
mkdir -p gpurun_out
for cfg in cfg3 cfg2 cfg3d cfg4 cfg5 cfg1; do
  steps=10; warm=3
  if [ "$cfg" = cfg5 ]; then steps=3; warm=3; fi
  timeout 900 python bench.py --config $cfg --steps $steps --warmup $warm > gpurun_out/${tag}_bench_${cfg}.json 2> gpurun_out/${tag}_bench_${cfg}.err
  echo "$cfg ours rc=$?"
  timeout 900 python bench.py --impl reference --config $cfg --steps 3 --warmup 1 > gpurun_out/${tag}_ref_${cfg}.json 2> gpurun_out/${tag}_ref_${cfg}.err
  echo "$cfg ref rc=$?"
done
