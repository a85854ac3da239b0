#!/bin/bash
# tensor-core run kernel trial: parity tests with PNDF_TC=1 (short timeouts), then config-5 A/B
mkdir -p gpurun_out
PNDF_TC=1 timeout ${TT:-400} python -m pytest tests/test_gpu_parity.py -q -x ${PYTEST_ARGS} > gpurun_out/pytest_tc.log 2>&1; echo rc=$? >> gpurun_out/pytest_tc.log
tail -4 gpurun_out/pytest_tc.log
if [ -z "$NOBENCH" ]; then
NOTEST=1 ENVS="${ENVS:-tc:PNDF_TC=1 base:}" bash tools/gpurun/ab_env.sh
fi
