#!/bin/bash
# A/B of the split hash (LIBS="name=path ..."): one-row steps through the C ABI and the device loop.
for L in ${LIBS}; do
  echo "== ${L%%=*}"; RG_LIB_PATH=${L#*=} timeout 200 python scripts/ab_split.py | grep "n=10000\|n=1000:"
  RG_LIB_PATH=${L#*=} timeout 300 python scripts/device_loop_diag.py 2>&1 | grep "device_loop=1" | cut -c1-100
done
