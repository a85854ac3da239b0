#!/bin/bash
# e2e chunk-count A/B on config 5 (PNDF_E2E_CHUNKS; default 8)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 3"
for k in 8 4 6 12 16; do PNDF_E2E_CHUNKS=$k timeout 600 $B > gpurun_out/e2e_$k.log 2>&1; done
