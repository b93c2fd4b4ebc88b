#!/bin/bash
# A/B: the two-step rollout's cp.async ring depth (slot pairs in flight) on C2, via library
# variants (RG_LIB_PATH); then the GPU kernel tests on the deeper ring.
mkdir -p gpurun_out
for r in 1 2 3; do
for L in base=paper_2510_08288_b200/_lib/librefgov_b200.so rp3=paper_2510_08288_b200/_lib/variants/rp3/librefgov_b200.so; do
  name=${L%%=*}; path=${L#*=}
  RG_LIB_PATH=$path timeout 300 python bench.py --no-cpu-baseline --no-sweep --steps 2000 > gpurun_out/ab_ring_$name.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/ab_ring_$name.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('$name', 'ms/step %.4f'%d['ms_per_step'] if d else 'FAILED '+open('gpurun_out/ab_ring_$name.log').read()[-600:], 'e2e %.4f'%d['e2e']['ms_per_step'] if d else '', 'span', d['latency']['k_grid_span_us'] if d else '', 'sm_mhz', d['clocks']['sm_mhz'] if d else '')"
done
done
RG_LIB_PATH=paper_2510_08288_b200/_lib/variants/rp3/librefgov_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/ab_ring_tests.log 2>&1; echo "rp3 tests rc=$?"; tail -2 gpurun_out/ab_ring_tests.log
