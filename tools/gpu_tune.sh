#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for rep in 1 2; do
    for c in 5 4; do
    timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/ab_${c}_$rep.log 2>&1
    echo "c$c $rep $(grep -o '"value": [0-9.e+]*' gpurun_out/ab_${c}_$rep.log | head -1) $(grep -o '"kernel_ms": [0-9.e+]*' gpurun_out/ab_${c}_$rep.log | head -1) $(grep -o '"pass": [a-z]*' gpurun_out/ab_${c}_$rep.log | head -1)" >> gpurun_out/ab.txt
    done
done
