#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "shards_bitwise" > gpurun_out/pytest_shardbits.log 2>&1; echo rc=$? >> gpurun_out/pytest_shardbits.log
