#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sampler.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for rep in 1 2; do
  for v in libpndf libpndf_sb0; do
    PNDF_LIB=paper_2109_14807_b200/$v.so timeout 600 python bench.py --op sample --no-cpu-baseline > gpurun_out/abs_${v}_$rep.log 2>&1
    echo "sample $v $rep $(grep -o '"value": [0-9.e+]*' gpurun_out/abs_${v}_$rep.log | head -1)" >> gpurun_out/ab.txt
  done
done
