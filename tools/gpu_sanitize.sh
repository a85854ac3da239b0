#!/bin/bash
# compute-sanitizer memcheck (one tool per call) on the smoke test and a parity subset
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests -m gpu -x -q -k "edge_cases or random_store_parity and N16_s1_L5_A5 or store_image or sampler_blank or binning_sorts_by_half_cell_key and 3 or tiled_query_parity and 2 or sg_rects and 2" > gpurun_out/memcheck.log 2>&1
echo rc=$? >> gpurun_out/memcheck.log
