#!/bin/bash
# e2e chunking A/B on config 5: chunk count x queries-per-row floor of a binned chunk
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 3"
for cfg in "16 4" "16 2" "32 2" "24 3" "64 1"; do set -- $cfg
  PNDF_E2E_CHUNKS=$1 PNDF_E2E_MINQ=$2 timeout 600 $B > gpurun_out/e2e2_$1_$2.log 2>&1; done
