#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wang.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --op wang > gpurun_out/bench_wang.log 2>&1
TCMD="python bench.py --op wang --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiled_query -c 1 -o gpurun_out/prof_tiled -f $TCMD > gpurun_out/ncu_tiled.log 2>&1
