#!/bin/bash
# parity first, then configs 5/4 timing (SAT format AUTO vs forced HILO via env)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
summ() { python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1),'Mq/s step', round(d['ms_per_step'],2),'ms query', round(d['roofline']['kernel_ms'],2),'bin',round(d['roofline']['binning_ms'],2), 'parity', d.get('parity_sample'))"; }
for c in 5 4 2; do
  echo "== config $c" >> gpurun_out/tune.log
  timeout 400 python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | summ >> gpurun_out/tune.log 2>&1
  echo "== config $c HILO" >> gpurun_out/tune.log
  PNDF_PREFIX=hilo timeout 400 python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | summ >> gpurun_out/tune.log 2>&1
done
