#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sampler.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --op sample > gpurun_out/bench_sample.log 2>&1
SCMD="python bench.py --op sample --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sample_kernel -c 1 -o gpurun_out/prof_sample -f $SCMD > gpurun_out/ncu_sample.log 2>&1
