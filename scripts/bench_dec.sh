#!/bin/bash
# A/B: grid-step kernels (0 per-step, 1 block-phased decoupled, 2 warp-specialised)
for K in ${KERNELS:-0 2}; do
  for N in ${NS:-1000 10000 100000}; do
    RG_GRID_KERNEL=$K timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-sweep --e2e-steps 5 --n-sim $N > gpurun_out/dec.log 2>&1
    python -c "
import json
l=[x for x in open('gpurun_out/dec.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('KERNEL=$K N=$N', 'ms/step %.4f'%d['ms_per_step'] if d else 'FAILED '+open('gpurun_out/dec.log').read()[-400:], 'G/s %.1f'%(d['value']/1e9) if d else '')"
  done
done
