#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
summ() { python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d.get('parity_sample') or {}; print(round(d['value']/1e6,1),'Mq/s step', round(d['ms_per_step'],2),'ms query', round(d['roofline']['kernel_ms'],2),'bin',round(d['roofline']['binning_ms'],2), 'parity', p.get('pass'), p.get('max_rel_err_nonzero'), 'e2e', (d.get('e2e') or {}).get('value'))"; }
for lib in libpndf.so libpndf_notma.so; do
  for c in 5 4; do
    echo "== $lib config $c" >> gpurun_out/tune.log
    PNDF_LIB=$PWD/paper_2109_14807_b200/$lib timeout 400 python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | summ >> gpurun_out/tune.log 2>&1
  done
  echo "== $lib config 5 HILO" >> gpurun_out/tune.log
  PNDF_PREFIX=hilo PNDF_LIB=$PWD/paper_2109_14807_b200/$lib timeout 400 python bench.py --config 5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | summ >> gpurun_out/tune.log 2>&1
done
