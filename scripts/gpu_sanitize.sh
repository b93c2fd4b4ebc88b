#!/bin/bash
# One compute-sanitizer tool per gpurun call (B200_PROFILING.md).  Small cases only.
TOOL=${1:-memcheck}
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool $TOOL --error-exitcode 99 python -m pytest -q -x -m gpu \
  -p no:cacheprovider "tests/test_gpu_parity.py::test_fill_cells_bit_exact" \
  "tests/test_gpu_kernels.py::test_bisect_both_rng_paths" \
  "tests/test_gpu_kernels.py::test_batch_every_lane_split" \
  "tests/test_gpu_parity.py::test_repeated_steps_reset_device_accumulators" \
  > gpurun_out/sanitize_$TOOL.log 2>&1
echo "sanitizer rc=$?" >> gpurun_out/sanitize_$TOOL.log
tail -6 gpurun_out/sanitize_$TOOL.log
