#!/bin/bash
mkdir -p gpurun_out
for v in libpndf_r32 libpndf_w32; do
PNDF_LIB=paper_2109_14807_b200/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "binning or binned" > gpurun_out/pytest_$v.log 2>&1; echo rc=$? >> gpurun_out/pytest_$v.log
done
for rep in 1 2; do
  for v in libpndf libpndf_r24 libpndf_r32 libpndf_w32; do
    PNDF_LIB=paper_2109_14807_b200/$v.so timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab_${v}_$rep.log 2>&1
    echo "c5 $v $rep $(grep -o '"value": [0-9.e+]*' gpurun_out/ab_${v}_$rep.log | head -1) $(grep -o '"binning_ms": [0-9.e+]*' gpurun_out/ab_${v}_$rep.log | head -1)" >> gpurun_out/ab.txt
  done
done
