#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --op wang > gpurun_out/bench_wang.log 2>&1; echo rc=$? >> gpurun_out/bench_wang.log
timeout 600 python bench.py --op wang_sample > gpurun_out/bench_wang_sample.log 2>&1; echo rc=$? >> gpurun_out/bench_wang_sample.log
