#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "sg or wang" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --op sg > gpurun_out/bench_sg.log 2>&1; echo rc=$? >> gpurun_out/bench_sg.log
timeout 900 python bench.py --op wang > gpurun_out/bench_wang.log 2>&1; echo rc=$? >> gpurun_out/bench_wang.log
