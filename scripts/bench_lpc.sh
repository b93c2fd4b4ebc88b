#!/bin/bash
for L in 1 2 4; do
  for N in 1000 4000 10000; do
    RG_FORCE_LPC=$L timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-sweep --e2e-steps 20 --n-sim $N > gpurun_out/lpc_${L}_${N}.log 2>&1
    python -c "
import json,sys
l=[x for x in open('gpurun_out/lpc_${L}_${N}.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('LPC=$L N=$N', 'ms/step %.4f'%d['ms_per_step'] if d else 'FAILED', 'G/s %.1f'%(d['value']/1e9) if d else '')"
  done
done
