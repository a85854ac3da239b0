#!/bin/bash
# binning kernels of config 5: launch list (per-kernel time) and one full capture of the scatter pass
mkdir -p gpurun_out
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bin.csv $SMALL > gpurun_out/ncu_launches_bin.log 2>&1
echo rc=$? >> gpurun_out/ncu_launches_bin.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rs_scatter -s 3 -c 1 -o gpurun_out/prof_scatter2 $SMALL > gpurun_out/ncu_scatter2.log 2>&1
echo rc=$? >> gpurun_out/ncu_scatter2.log
