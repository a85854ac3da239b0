#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for rep in 1 2; do
  for v in libpndf libpndf_pf0; do
    for c in 5 4; do
    PNDF_LIB=paper_2109_14807_b200/$v.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/ab_${v}_${c}_$rep.log 2>&1
    echo "c$c $v $rep $(grep -o '"value": [0-9.e+]*' gpurun_out/ab_${v}_${c}_$rep.log | head -1) $(grep -o '"kernel_ms": [0-9.e+]*' gpurun_out/ab_${v}_${c}_$rep.log | head -1) $(grep -o '"pass": [a-z]*' gpurun_out/ab_${v}_${c}_$rep.log | head -1)" >> gpurun_out/ab.txt
    done
  done
done
