#!/bin/bash
mkdir -p gpurun_out
for g in 0 8 4 2 1; do timeout 400 python bench.py --op wang_sample --lanes $g > gpurun_out/wlanes_$g.log 2>&1; done
for g in 0 4 2; do timeout 400 python bench.py --op wang --lanes $g > gpurun_out/wqlanes_$g.log 2>&1; done
