#!/bin/bash
# A/B of the radix-scatter CTA size on config 5 (binning time) + the binning tests under both
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/ab_256.log 2>&1
PNDF_SCATTER_THREADS=512 timeout 300 $B > gpurun_out/ab_512.log 2>&1
PNDF_SCATTER_THREADS=512 timeout 900 python -m pytest tests -m gpu -x -q -k "bin or parity" > gpurun_out/pytest_512.log 2>&1; echo rc=$? >> gpurun_out/pytest_512.log
