#!/bin/bash
mkdir -p gpurun_out
./tools/membw > gpurun_out/membw.json 2>&1 || (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membw tools/membw.cu && ./tools/membw > gpurun_out/membw.json 2>&1)
for b in off on; do
  CMD="python bench.py --queries 100000000 --bin $b --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  timeout 600 $CMD > gpurun_out/plain_$b.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:query_kernel -c 1 -o gpurun_out/prof_c5_$b $CMD > gpurun_out/ncu_$b.log 2>&1
  echo rc=$? >> gpurun_out/ncu_$b.log
done
