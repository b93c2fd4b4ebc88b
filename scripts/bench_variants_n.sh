#!/bin/bash
# A/B of library builds at several scenario counts: device ms/step
for so in "$@"; do
  for N in 1000 10000 100000; do
    RG_LIB_PATH=$so timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-sweep --e2e-steps 5 --n-sim $N > gpurun_out/varn.log 2>&1
    python -c "
import json,os
l=[x for x in open('gpurun_out/varn.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print(os.path.basename('$so'), 'N=$N', 'ms/step %.4f'%d['ms_per_step'] if d else 'FAILED', 'G/s %.1f'%(d['value']/1e9) if d else open('gpurun_out/varn.log').read()[-300:])"
  done
done
