#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --config 1 > gpurun_out/bench_c1.log 2>&1; echo rc=$? >> gpurun_out/bench_c1.log
timeout 300 python bench.py --config 2 > gpurun_out/bench_c2.log 2>&1; echo rc=$? >> gpurun_out/bench_c2.log
