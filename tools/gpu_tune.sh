#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_als.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_als.csv python bench.py --op als --config 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_als_l.log 2>&1
timeout 600 python bench.py --op als --config 2 > gpurun_out/bench_als.log 2>&1
