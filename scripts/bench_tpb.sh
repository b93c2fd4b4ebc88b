#!/bin/bash
# occupancy probe: ms/step vs scenario count and block size (RG_FORCE_TPB)
for T in ${TPBS:-32 64 128}; do
  for N in ${NS:-1000}; do
    RG_FORCE_TPB=$T timeout 300 python bench.py --steps ${STEPS:-200} --warmup 5 --no-cpu-baseline --no-sweep --e2e-steps 5 --n-sim $N > gpurun_out/tpb.log 2>&1
    python -c "
import json
l=[x for x in open('gpurun_out/tpb.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('TPB=$T N=$N', 'ms/step %.4f'%d['ms_per_step'] if d else 'FAILED '+open('gpurun_out/tpb.log').read()[-300:], 'G/s %.1f'%(d['value']/1e9) if d else '')"
  done
done
