#!/bin/bash
# A/B pass: micro rollout probe, GPU tests on the default build, bench of the default build
# against the library variants given as arguments (RG_LIB_PATH).
mkdir -p gpurun_out
[ -x scripts/micro/rollout_occ ] && timeout 120 ./scripts/micro/rollout_occ > gpurun_out/occ.txt 2>&1
[ -n "$NOTEST" ] || PYTEST_TIMEOUT=600 bash scripts/gpu_tests.sh
for so in paper_2510_08288_b200/_lib/librefgov_b200.so "$@"; do
  tag=$(basename $so .so)
  RG_LIB_PATH=$so timeout 400 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline \
    --e2e-steps 200 > gpurun_out/ab_$tag.log 2>&1
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
l = [x for x in open(f"gpurun_out/ab_{tag}.log") if x.startswith('{')]
if not l:
    print(tag, "FAILED"); print(open(f"gpurun_out/ab_{tag}.log").read()[-1500:]); sys.exit()
d = json.loads(l[0])
sw = [(s.get('n_sim') or s.get('workload')[:30], round(s['ms_per_step'], 4)) for s in d['sweep']]
print(tag, "ms/step %.4f p50 %.4f" % (d['ms_per_step'], d['kernel_ms_p50']),
      "e2e %.4f" % d['e2e']['ms_per_step'], sw)
PY
done
