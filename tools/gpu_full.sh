#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/full_1.log 2>&1
PNDF_SCATTER_FULL=0 timeout 300 $B > gpurun_out/full_0.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "bin or parity or shard" > gpurun_out/pytest_full.log 2>&1; echo rc=$? >> gpurun_out/pytest_full.log
