#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wang.py -x -q > gpurun_out/pytest_wang.log 2>&1; echo rc=$? >> gpurun_out/pytest_wang.log
timeout 600 python bench.py --op wang > gpurun_out/bench_wang.log 2>&1; echo rc=$? >> gpurun_out/bench_wang.log
