#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_bin2.log 2>&1; echo rc=$? >> gpurun_out/b_bin2.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bin2.csv $SMALL > gpurun_out/ncu_launches_bin2.log 2>&1
