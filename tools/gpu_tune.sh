#!/bin/bash
# per-GPU cost of the 2/4/8-GPU config-5 jobs on one GPU: shard 0 of W, spatial vs index sharding
mkdir -p gpurun_out
for w in 2 4 8; do
  for sh in spatial index; do
    timeout 900 python bench.py --as-shard 0/$w --shard $sh --no-e2e --no-cpu-baseline > gpurun_out/as_${sh}_$w.log 2>&1
    echo "W=$w $sh $(grep -o '"value": [0-9.e+]*' gpurun_out/as_${sh}_$w.log | head -1) $(grep -o '"ms_per_step": [0-9.e+]*' gpurun_out/as_${sh}_$w.log | head -1) $(grep -o '"queries_per_rank": [0-9]*' gpurun_out/as_${sh}_$w.log | head -1) $(grep -o '"pass": [a-z]*' gpurun_out/as_${sh}_$w.log | head -1)" >> gpurun_out/as.txt
  done
done
