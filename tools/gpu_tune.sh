#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "blocked" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --op blocked --config 2 > gpurun_out/bench_blocked.log 2>&1; echo rc=$? >> gpurun_out/bench_blocked.log
