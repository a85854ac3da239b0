#!/bin/bash
mkdir -p gpurun_out
C="python bench.py --op wang_sample --steps 1 --warmup 1"
timeout 600 $C > gpurun_out/plain_wsample.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiled_sample -c 1 -o gpurun_out/prof_tsample2 -f $C > gpurun_out/ncu_tsample2.log 2>&1
echo rc=$? >> gpurun_out/ncu_tsample2.log
Q="python bench.py --op wang --steps 1 --warmup 1"
timeout 600 $Q > gpurun_out/plain_wquery.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiled_query -c 1 -o gpurun_out/prof_tquery2 -f $Q > gpurun_out/ncu_tquery2.log 2>&1
echo rc=$? >> gpurun_out/ncu_tquery2.log
