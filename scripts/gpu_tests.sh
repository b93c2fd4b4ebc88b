#!/bin/bash
# GPU-side test run used with gpurun: logs land in gpurun_out/ as they are written.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_info.txt 2>&1
grep -o -w -E "fma|avx2|avx512f" /proc/cpuinfo | sort | uniq -c >> gpurun_out/gpu_info.txt
nproc >> gpurun_out/gpu_info.txt
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q -p no:cacheprovider \
  -o faulthandler_timeout=300 "$@" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log
