#!/bin/bash
# GPU test suite + smoke (round-end equivalent); logs in gpurun_out/
mkdir -p gpurun_out
timeout ${T:-2400} python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
