#!/bin/bash
mkdir -p gpurun_out
bash tools/gpurun/tests_gpu.sh
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity"
timeout 600 $CMD > gpurun_out/plain_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:query_g4 -c 1 -o gpurun_out/prof_query_full -f $CMD > gpurun_out/ncu_full.log 2>&1
echo full_rc=$? >> gpurun_out/ncu_full.log
