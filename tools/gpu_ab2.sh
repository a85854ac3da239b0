#!/bin/bash
# A/B: radix-scatter value loads after the ranking (PNDF_SCATTER_LATEV=1) vs with the keys; then the
# per-GPU cost of the 2/4/8-GPU spatial shards of config 5 on one GPU (--as-shard)
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/ab2_base.log 2>&1
PNDF_SCATTER_LATEV=1 timeout 300 $B > gpurun_out/ab2_latev.log 2>&1
for w in 2 4 8; do timeout 300 $B --as-shard 0/$w > gpurun_out/shard_$w.log 2>&1; done
