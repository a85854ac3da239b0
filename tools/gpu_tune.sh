#!/bin/bash
mkdir -p gpurun_out
summ() { python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d.get('parity_sample') or {}; print(round(d['value']/1e6,1),'Mq/s step', round(d['ms_per_step'],2),'ms query', round(d['roofline']['kernel_ms'],2),'bin',round(d['roofline'].get('binning_ms',0),2))"; }
for lib in libpndf.so libpndf_zna0.so libpndf_base.so; do
  for c in 5 4; do
  echo "== $lib config $c" >> gpurun_out/tune.log
  PNDF_LIB=$PWD/paper_2109_14807_b200/$lib timeout 400 python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-parity 2>&1 | summ >> gpurun_out/tune.log 2>&1
done; done
