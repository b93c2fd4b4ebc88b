#!/bin/bash
# A/B: time-split chunk size / slots (LIBS="name=path ..."): parity subset, C1, 1k/10k one-row steps, C3.
for L in ${LIBS}; do
  echo "== ${L%%=*}"
  RG_LIB_PATH=${L#*=} timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_native_loop.py -x -q -p no:cacheprovider -k "time_split or device or c1 or bisection" 2>&1 | tail -1
  RG_LIB_PATH=${L#*=} timeout 300 python scripts/c1_steady.py
  RG_LIB_PATH=${L#*=} timeout 200 python scripts/ab_split.py | grep "n=1000:\|n=10000"
  RG_LIB_PATH=${L#*=} timeout 300 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/ch.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/ch.json') if l.startswith('{')][-1]); print('c3 ms/step %.5f' % d['ms_per_step'])"
done
