#!/bin/bash
# ncu --set full of the query kernel (ring or plain with PNDF_NORING=1), config 5 full batch
mkdir -p gpurun_out
TAG=${TAG:-ring}; K=${K:-query_ring}
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity"
timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo rc=$? >> gpurun_out/ncu_$TAG.log; tail -2 gpurun_out/ncu_$TAG.log
