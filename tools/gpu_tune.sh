#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
  for v in libpndf libpndf_f20; do
    PNDF_LIB=paper_2109_14807_b200/$v.so timeout 600 python bench.py --config 4 --no-e2e --no-cpu-baseline > gpurun_out/ab4_${v}_$rep.log 2>&1
    echo "c4 $v $rep $(grep -o '"value": [0-9.e+]*' gpurun_out/ab4_${v}_$rep.log | head -1) $(grep -o '"kernel_ms": [0-9.e+]*' gpurun_out/ab4_${v}_$rep.log | head -1)" >> gpurun_out/ab.txt
    PNDF_LIB=paper_2109_14807_b200/$v.so timeout 600 python bench.py --config 3 --no-e2e --no-cpu-baseline > gpurun_out/ab3_${v}_$rep.log 2>&1
    echo "c3 $v $rep $(grep -o '"value": [0-9.e+]*' gpurun_out/ab3_${v}_$rep.log | head -1) $(grep -o '"kernel_ms": [0-9.e+]*' gpurun_out/ab3_${v}_$rep.log | head -1)" >> gpurun_out/ab.txt
  done
done
