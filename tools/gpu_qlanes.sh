#!/bin/bash
# query-kernel lanes-per-query A/B on configs 2-4 (default: G = R/4 capped at 32, NV = 1)
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu-baseline"
for g in 0 4 2; do timeout 300 $B --config 2 --lanes $g > gpurun_out/q2_$g.log 2>&1; done
for g in 0 8 4; do timeout 400 $B --config 3 --lanes $g > gpurun_out/q3_$g.log 2>&1; done
for g in 0 16; do timeout 400 $B --config 4 --lanes $g > gpurun_out/q4_$g.log 2>&1; done
