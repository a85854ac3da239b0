#!/bin/bash
# parity tests of the default library, then config-5 bench of each library variant
# (VARIANTS="a b ..."; "base" = libpndf.so, NAME = libpndf_NAME.so from build.py --variant=NAME:DEFS)
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo rc=$? >> gpurun_out/pytest_parity.log
tail -2 gpurun_out/pytest_parity.log
fi
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${BARGS}"
for v in ${VARIANTS:-base}; do
  case $v in
    base) env="" ;;
    *) env="PNDF_LIB=$PWD/paper_2109_14807_b200/libpndf_$v.so" ;;
  esac
  env $env timeout 600 $B > gpurun_out/ab_$v.log 2>&1
  python - "$v" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/ab_{f}.log").read().strip().splitlines()[-1])
    r=d["roofline"]; ps=d.get("parity_sample") or {}
    print(f"{f:10s} value {d['value']:.3e} kernel_ms {r['kernel_ms']:.2f} bin_ms {r['binning_ms']:.2f} parity {ps.get('pass')} checksum {d['checksum']}")
except Exception as e:
    print(f, "ERR", e, open(f"gpurun_out/ab_{f}.log").read()[-1500:])
PY
done
