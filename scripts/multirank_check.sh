#!/bin/bash
# Functional check of bench.py's N-rank path at the headline config (ranks
# share the one GPU, gloo collectives; timings meaningless): the row-block
# split of cfg3's largest element at N=4 and the sharded compute_mapper e2e.
mkdir -p gpurun_out
B200MAP_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 4 --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/bench_n4_cfg3_gloo.log 2>&1; echo "n4 cfg3 gloo rc=$?"
tail -1 gpurun_out/bench_n4_cfg3_gloo.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nodes', d['nodes'], 'edges', d['edges'], 'n_gpus', d['n_gpus'])"
