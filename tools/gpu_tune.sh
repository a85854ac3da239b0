#!/bin/bash
mkdir -p gpurun_out
summ() { python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d.get('parity_sample') or {}; print(round(d['value']/1e6,1),'Mq/s step', round(d['ms_per_step'],2),'ms query', round(d['roofline']['kernel_ms'],2),'bin',round(d['roofline'].get('binning_ms',0),2), 'parity', p.get('pass'), p.get('max_rel_err_nonzero'))"; }
for sp in 1 2; do
  echo "== split $sp config 5" >> gpurun_out/tune.log
  PNDF_RANK_SPLIT=$sp timeout 400 python bench.py --config 5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | summ >> gpurun_out/tune.log 2>&1
  echo "== split $sp config 5 shard" >> gpurun_out/tune.log
  PNDF_RANK_SPLIT=$sp timeout 400 python bench.py --config 5 --queries 125000000 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | summ >> gpurun_out/tune.log 2>&1
done
PNDF_RANK_SPLIT=2 timeout 900 python -m pytest tests -m gpu -x -q -k "config5 or random_store or lane_splits" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
