#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --op sweep > gpurun_out/bench_sweep.log 2>&1; echo rc=$? >> gpurun_out/bench_sweep.log
