#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --config 3 --s0 4 > gpurun_out/bench_c3_s04.log 2>&1; echo rc=$? >> gpurun_out/bench_c3_s04.log
timeout 600 python bench.py --config 3 --s0 4 --bin on --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_s04_bin.log 2>&1; echo rc=$? >> gpurun_out/bench_c3_s04_bin.log
