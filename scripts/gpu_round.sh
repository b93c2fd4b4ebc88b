#!/bin/bash
# Full GPU pass used during development: tests + smoke, bench / reference arm / launch list /
# ncu summaries (scripts/gpu_profiles.sh, keeps gpurun_out/ small), N=2 smoke over gloo.
mkdir -p gpurun_out
PYTEST_TIMEOUT=800 bash scripts/gpu_tests.sh
TAG=${TAG:-r} bash scripts/gpu_profiles.sh
RG_BENCH_DIST_BACKEND=gloo RG_BENCH_DEVICE=0 timeout 300 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 \
  --warmup 3 --e2e-steps 5 --no-sweep > gpurun_out/bench_n2_smoke.log 2>&1
echo "n2 smoke rc=$?"; grep -o '"value": [0-9.e+]*' gpurun_out/bench_n2_smoke.log | head -2
