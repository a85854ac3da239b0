#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_wang.py -x -q > gpurun_out/pytest_sampler.log 2>&1; echo rc=$? >> gpurun_out/pytest_sampler.log
timeout 600 python bench.py --op sample > gpurun_out/bench_sample.log 2>&1
timeout 600 python bench.py --op sample --config 2 > gpurun_out/bench_sample_c2.log 2>&1
timeout 600 python bench.py --op sample --config 1 > gpurun_out/bench_sample_c1.log 2>&1
timeout 600 python bench.py --op sample --config 1 --lanes 8 > gpurun_out/bench_sample_c1_l8.log 2>&1
