#!/bin/bash
# A/B: k_grid_pairs register cap (launch bounds 128 x MINB) on C5, via library variants.
mkdir -p gpurun_out
for r in 1 2; do
for L in base=paper_2510_08288_b200/_lib/librefgov_b200.so lb4=paper_2510_08288_b200/_lib/variants/lb4/librefgov_b200.so lb5=paper_2510_08288_b200/_lib/variants/lb5/librefgov_b200.so lb6=paper_2510_08288_b200/_lib/variants/lb6/librefgov_b200.so lb8=paper_2510_08288_b200/_lib/variants/lb8/librefgov_b200.so; do
  name=${L%%=*}; path=${L#*=}
  RG_LIB_PATH=$path timeout 600 python bench.py --workload c5 --no-cpu-baseline --no-sweep > gpurun_out/ab_c5_$name.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/ab_c5_$name.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('$name', 'ms/step %.2f'%d['ms_per_step'] if d else 'FAILED '+open('gpurun_out/ab_c5_$name.log').read()[-600:], 'value %.4g'%d['value'] if d else '', 'roof', d.get('roofline',{}).get('frac') if d else '', 'sm_mhz', d['clocks']['sm_mhz'] if d else '')"
done
done
