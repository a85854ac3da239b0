#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_als.py -q > gpurun_out/als3.log 2>&1; echo rc=$? >> gpurun_out/als3.log
timeout 900 python bench.py --op als --config 2 > gpurun_out/bench_als.log 2>&1; echo rc=$? >> gpurun_out/bench_als.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_als.csv python bench.py --op als --config 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_als_l.log 2>&1; echo rc=$? >> gpurun_out/ncu_als_l.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mttkrp_gemm -s 6 -c 2 -o gpurun_out/prof_als -f python bench.py --op als --config 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_als.log 2>&1; echo rc=$? >> gpurun_out/ncu_als.log
