#!/bin/bash
# A/B: the speculative true-plant step in the device loop (LIBS="name=path ...").
timeout 600 python -m pytest tests/test_gpu_native_loop.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "native or device or closed_loop or transient_golden or large" 2>&1 | tail -1
for r in 1 2; do for L in ${LIBS}; do
  echo "== ${L%%=*}"
  RG_LIB_PATH=${L#*=} timeout 300 python scripts/device_loop_diag.py 2>&1 | grep "device_loop=1" | cut -c1-70
  RG_LIB_PATH=${L#*=} timeout 300 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/sp.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/sp.json') if l.startswith('{')][-1]); print('c3 ms/step %.5f' % d['ms_per_step'])"
done; done
