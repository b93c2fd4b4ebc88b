#!/bin/bash
# quick A/B of library builds: device step time at the bench workload
for so in "$@"; do
  RG_LIB_PATH=$so timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --e2e-steps 50 > gpurun_out/var_$(basename $so).log 2>&1
  python - "$so" <<'PY'
import json,sys
so=sys.argv[1]; import os
l=[x for x in open(f"gpurun_out/var_{os.path.basename(so)}.log") if x.startswith('{')]
if not l: print(so, "FAILED"); print(open(f"gpurun_out/var_{os.path.basename(so)}.log").read()[-800:]); sys.exit()
d=json.loads(l[0]); print(os.path.basename(so), "ms/step %.4f"%d['ms_per_step'], "frac %.3f"%d['roofline']['frac'])
PY
done
