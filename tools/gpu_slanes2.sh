#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wang.py -x -q > gpurun_out/pytest_wang.log 2>&1; echo rc=$? >> gpurun_out/pytest_wang.log
timeout 400 python bench.py --op wang_sample > gpurun_out/bench_wang_sample.log 2>&1
for g in 0 1 2 4; do timeout 400 python bench.py --op sample --config 2 --lanes $g > gpurun_out/s2lanes_$g.log 2>&1; done
for g in 0 2 4; do timeout 400 python bench.py --op sample --config 4 --lanes $g > gpurun_out/s4lanes_$g.log 2>&1; done
