#!/bin/bash
# parity (main lib) then variant sweep on configs 5/4/2 (+ config 5 at the 8-GPU shard size)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
summ() { python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d.get('parity_sample') or {}; print(round(d['value']/1e6,1),'Mq/s step', round(d['ms_per_step'],2),'ms query', round(d['roofline']['kernel_ms'],2),'bin',round(d['roofline']['binning_ms'],2), 'parity', p.get('pass'), p.get('max_rel_err_nonzero'), 'e2e', (d.get('e2e') or {}).get('value'))"; }
for lib in libpndf.so libpndf_k4m1.so libpndf_k4m2.so libpndf_k8m1.so; do
  for c in 5 4 2; do
    echo "== $lib config $c" >> gpurun_out/tune.log
    PNDF_LIB=$PWD/paper_2109_14807_b200/$lib timeout 400 python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | summ >> gpurun_out/tune.log 2>&1
  done
done
for b in on off; do
  echo "== config 5 shard 125M bin=$b" >> gpurun_out/tune.log
  timeout 400 python bench.py --queries 125000000 --bin $b --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | summ >> gpurun_out/tune.log 2>&1
done
echo "== config 5 e2e" >> gpurun_out/tune.log
timeout 400 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | summ >> gpurun_out/tune.log 2>&1
