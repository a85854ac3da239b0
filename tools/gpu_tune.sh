#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blocked.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --op blocked --config 2 > gpurun_out/bench_blocked.log 2>&1
BCMD="python bench.py --op blocked --config 2 --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:blocked_query -c 1 -o gpurun_out/prof_blocked -f $BCMD > gpurun_out/ncu_blocked.log 2>&1
