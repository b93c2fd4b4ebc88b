#!/bin/bash
# A/B: one-unit tanh-batch placement (LIBS="name=path ..."): C1 loop, 1k one-row steps, device loop.
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_native_loop.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "time_split or native or device or c1 or bisection or transient_golden" 2>&1 | tail -1
for r in 1 2; do for L in ${LIBS}; do
  echo "== ${L%%=*}"; RG_LIB_PATH=${L#*=} timeout 300 python scripts/c1_steady.py
  RG_LIB_PATH=${L#*=} timeout 200 python scripts/ab_split.py | grep "n=1000:\|n=4000"
  RG_LIB_PATH=${L#*=} timeout 300 python scripts/device_loop_diag.py 2>&1 | grep "n=1000 device_loop=1" | cut -c1-60
done; done
