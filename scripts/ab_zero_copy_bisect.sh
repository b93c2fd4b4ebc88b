#!/bin/bash
# Zero-copy results of rg_bisect and the persistent joint search: the bisection/joint tests,
# then the C-ABI call times (LIBS="name=path ...").
timeout 900 python -m pytest tests/test_gpu_joint.py tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "bisect or joint or probe or sequential or alg2 or c1 or c4_1m_seq" 2>&1 | tail -2
for L in ${LIBS}; do
  echo "== ${L%%=*}"
  RG_LIB_PATH=${L#*=} timeout 300 python scripts/ab_bisect_probe.py 2>&1 | grep "steady" | cut -c1-110
  RG_LIB_PATH=${L#*=} timeout 300 python scripts/ab_joint_probe.py 2>&1 | grep "steady\|transient" | cut -c1-110
done
