#!/bin/bash
# ncu --set full capture of one radix scatter pass (config 5, 1e9 queries)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-rs_scatter} -s ${SKIP:-1} -c 1 -o gpurun_out/prof_${PNAME:-scatter} -f $CMD > gpurun_out/ncu_scatter.log 2>&1
echo scatter_rc=$? >> gpurun_out/ncu_scatter.log; tail -1 gpurun_out/ncu_scatter.log
