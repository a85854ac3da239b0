#!/bin/bash
# parity first, then binning on/off on configs 3-5 (+ kernel occupancy variants on config 5)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
summ() { python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1),'Mq/s step', round(d['ms_per_step'],2),'ms query', round(d['roofline']['kernel_ms'],2),'bin',round(d['roofline']['binning_ms'],2))"; }
for lib in libpndf.so libpndf_minb1.so libpndf_minb3.so; do for b in on off; do
  echo "== config 5 $lib bin=$b" >> gpurun_out/tune.log
  PNDF_LIB=$PWD/paper_2109_14807_b200/$lib timeout 300 python bench.py --config 5 --bin $b --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | summ >> gpurun_out/tune.log 2>&1
done; done
for c in 4 3; do for b in on off; do
  echo "== config $c bin=$b" >> gpurun_out/tune.log
  timeout 300 python bench.py --config $c --bin $b --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | summ >> gpurun_out/tune.log 2>&1
done; done
