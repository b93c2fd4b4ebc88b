for r in 1 2 3; do
for L in sp1=paper_2510_08288_b200/_lib/librefgov_b200.so sp3=paper_2510_08288_b200/_lib/variants/sp3/librefgov_b200.so; do
  RG_LIB_PATH=${L#*=} timeout 300 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/sp.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/sp.json') if l.startswith('{')][-1]); print('${L%%=*}', 'c3 ms/step %.5f' % d['ms_per_step'])"
done; done
