#!/bin/bash
# Full GPU pass used during development: tests, bench, launch list, N=2 smoke, reference arm.
mkdir -p gpurun_out
PYTEST_TIMEOUT=800 bash scripts/gpu_tests.sh
bash scripts/gpu_measure.sh ${TAG:-r}
SMALL="--steps 20 --warmup 3 --no-cpu-baseline --no-sweep --e2e-steps 5"
timeout 300 python bench.py $SMALL > gpurun_out/launch_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py $SMALL > gpurun_out/launch_ncu.log 2>&1
echo "launch list rc=$?"
RG_BENCH_DIST_BACKEND=gloo RG_BENCH_DEVICE=0 timeout 300 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 \
  --warmup 3 --e2e-steps 5 --no-sweep > gpurun_out/bench_n2_smoke.log 2>&1
echo "n2 smoke rc=$?"; grep -o '"value": [0-9.e+]*' gpurun_out/bench_n2_smoke.log | head -2
timeout 300 python bench.py --impl reference --cpu-seconds 5 > gpurun_out/bench_ref.log 2>&1
echo "reference rc=$?"; tail -c 600 gpurun_out/bench_ref.log
