#!/bin/bash
# ring-staged query kernel: parity tests, then config-5 bench A/B against query_kernel (PNDF_NORING=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo rc=$? >> gpurun_out/pytest_parity.log
tail -3 gpurun_out/pytest_parity.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/ring_on.log 2>&1
PNDF_NORING=1 timeout 600 $B > gpurun_out/ring_off.log 2>&1
for f in ring_on ring_off; do python - "$f" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/{f}.log").read().strip().splitlines()[-1])
    print(f, "value %.3e"%d["value"], "kernel_ms %.2f"%d["roofline"]["kernel_ms"], "bin_ms %.2f"%d["roofline"]["binning_ms"], "parity", d["parity_sample"]["pass"], d["checksum"])
except Exception as e:
    print(f, "ERR", e, open(f"gpurun_out/{f}.log").read()[-1500:])
PY
done
