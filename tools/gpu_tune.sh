#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
  for v in libpndf libpndf_w48; do
    PNDF_LIB=paper_2109_14807_b200/$v.so timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab_${v}_5_$rep.log 2>&1
    echo "c5 $v $rep $(grep -o '"value": [0-9.e+]*' gpurun_out/ab_${v}_5_$rep.log | head -1)" >> gpurun_out/ab.txt
    PNDF_LIB=paper_2109_14807_b200/$v.so timeout 600 python bench.py --op sg --no-cpu-baseline > gpurun_out/ab_${v}_sg_$rep.log 2>&1
    echo "sg $v $rep $(grep -o '"value": [0-9.e+]*' gpurun_out/ab_${v}_sg_$rep.log | head -1) $(grep -o '"pass": [a-z]*' gpurun_out/ab_${v}_sg_$rep.log | head -1)" >> gpurun_out/ab.txt
  done
done
