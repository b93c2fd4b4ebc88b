#!/bin/bash
# Time-split grid step: parity against k_grid, then the 1-row and C3 timings.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "time_split or row_plan" \
  > gpurun_out/ts_tests.log 2>&1; echo "ts tests rc=$?" >> gpurun_out/ts_tests.log
tail -3 gpurun_out/ts_tests.log
