#!/bin/bash
# A/B of library variants on the default bench (config 5): PNDF_LIB selects the .so
mkdir -p gpurun_out
for rep in 1 2; do
  for v in libpndf libpndf_f20; do
    PNDF_LIB=paper_2109_14807_b200/$v.so timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab_${v}_$rep.log 2>&1
    echo "$v $rep $(grep -o '"value": [0-9.e+]*' gpurun_out/ab_${v}_$rep.log | head -1) $(grep -o '"kernel_ms": [0-9.e+]*' gpurun_out/ab_${v}_$rep.log | head -1)" >> gpurun_out/ab.txt
  done
done
timeout 600 python -m pytest tests -m gpu -x -q -k "parity" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
