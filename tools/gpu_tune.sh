#!/bin/bash
# config 5 at the 8-GPU shard size (1.25e8 queries) and at 2 GPUs (5e8), single GPU
mkdir -p gpurun_out
for q in 125000000 250000000 500000000; do
timeout 600 python bench.py --queries $q --no-e2e --no-cpu-baseline > gpurun_out/shard_$q.log 2>&1
echo "$q $(grep -o '"value": [0-9.e+]*' gpurun_out/shard_$q.log | head -1) $(grep -o '"kernel_ms": [0-9.e+]*' gpurun_out/shard_$q.log | head -1) $(grep -o '"binning_ms": [0-9.e+]*' gpurun_out/shard_$q.log | head -1)" >> gpurun_out/shard.txt
done
