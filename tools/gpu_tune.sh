#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
  for v in libpndf libpndf_nr2 libpndf_nr3 libpndf_nr4; do
    PNDF_LIB=paper_2109_14807_b200/$v.so timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab_${v}_$rep.log 2>&1
    echo "c5 $v $rep $(grep -o '"value": [0-9.e+]*' gpurun_out/ab_${v}_$rep.log | head -1) $(grep -o '"kernel_ms": [0-9.e+]*' gpurun_out/ab_${v}_$rep.log | head -1) $(grep -o '"pass": [a-z]*' gpurun_out/ab_${v}_$rep.log | head -1)" >> gpurun_out/ab.txt
  done
done
