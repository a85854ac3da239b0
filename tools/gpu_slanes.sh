#!/bin/bash
# sampler lanes-per-sample A/B on config 5 (G = 32 / 16 / 8 lanes, NV = 2 / 4 / 8 float4 per lane)
mkdir -p gpurun_out
for g in 32 16 8; do timeout 400 python bench.py --op sample --lanes $g --steps 3 --no-cpu-baseline > gpurun_out/slanes_$g.log 2>&1; done
