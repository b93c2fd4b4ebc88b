#!/bin/bash
# A/B: library variants (RG_LIB_PATH) at several scenario counts; LIBS="name=path ..."
for L in ${LIBS}; do
  name=${L%%=*}; path=${L#*=}
  for N in ${NS:-1000 10000 100000}; do
    RG_LIB_PATH=$path timeout 300 python bench.py --steps ${STEPS:-300} --warmup 5 --no-cpu-baseline --no-sweep --e2e-steps 5 --n-sim $N > gpurun_out/ab.log 2>&1
    python -c "
import json
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('$name N=$N', 'ms/step %.4f'%d['ms_per_step'] if d else 'FAILED '+open('gpurun_out/ab.log').read()[-400:], 'G/s %.1f'%(d['value']/1e9) if d else '', 'sm_mhz', d['clocks']['sm_mhz'] if d else '')"
  done
done
