#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --op sample --steps 3 --warmup 2 > gpurun_out/bench_sample.log 2>&1; echo rc=$? >> gpurun_out/bench_sample.log
timeout 600 python bench.py --op sample --config 2 --steps 3 --warmup 2 > gpurun_out/bench_sample_c2.log 2>&1; echo rc=$? >> gpurun_out/bench_sample_c2.log
