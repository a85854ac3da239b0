#!/bin/bash
# A/B of runtime switches on one library: ENVS="name1:VAR=1,VAR2=0 name2: ..." (empty = defaults);
# parity tests first unless NOTEST=1; config-5 bench (BARGS extra bench args) per setting
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x ${PYTEST_ARGS} > gpurun_out/pytest_parity.log 2>&1; echo rc=$? >> gpurun_out/pytest_parity.log
tail -3 gpurun_out/pytest_parity.log
fi
B="python bench.py --steps ${STEPS:-3} --warmup 3 --no-e2e --no-cpu-baseline ${BARGS}"
for spec in ${ENVS:-base:}; do
  name=${spec%%:*}; vars=${spec#*:}
  env ${vars//,/ } timeout 900 $B > gpurun_out/ab_$name.log 2>&1
  python - "$name" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/ab_{f}.log").read().strip().splitlines()[-1])
    r=d["roofline"]; ps=d.get("parity_sample") or {}
    print(f"{f:12s} value {d['value']:.3e} kernel_ms {r.get('kernel_ms')} bin_ms {r.get('binning_ms')} parity {ps.get('pass')} {ps.get('max_rel_err')}")
except Exception as e:
    print(f, "ERR", e, open(f"gpurun_out/ab_{f}.log").read()[-1500:])
PY
done
