#!/bin/bash
# A/B: environment variants at several scenario counts; ENVS="name:VAR=val,VAR2=val ..."
for E in ${ENVS}; do
  name=${E%%:*}; vars=${E#*:}
  for N in ${NS:-1000 10000}; do
    env ${vars//,/ } timeout 300 python bench.py --steps ${STEPS:-300} --warmup 5 --no-cpu-baseline --no-sweep --e2e-steps 5 --n-sim $N > gpurun_out/envab.log 2>&1
    python -c "
import json
l=[x for x in open('gpurun_out/envab.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('$name N=$N', 'ms/step %.4f'%d['ms_per_step'] if d else 'FAILED '+open('gpurun_out/envab.log').read()[-400:], 'G/s %.1f'%(d['value']/1e9) if d else '', 'e2e %.4f'%d['e2e']['ms_per_step'] if d else '')"
  done
done
