#!/bin/bash
mkdir -p gpurun_out
for g in 0 4 2 1; do timeout 400 python bench.py --op blocked --config 2 --lanes $g > gpurun_out/bl_$g.log 2>&1; done
