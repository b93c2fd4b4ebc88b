#!/bin/bash
# bench + one ncu --set full capture of k_grid at the bench workload (N=1000); logs in gpurun_out/
TAG=${1:-x}
mkdir -p gpurun_out
timeout 400 python bench.py --steps ${STEPS:-1000} --warmup 10 --cpu-seconds ${CPUS:-5} > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
tail -c 1500 gpurun_out/bench_$TAG.log | grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|"value": [0-9.e+]*' | head -5
if [ -n "$NCU" ]; then
  python scripts/prof_grid.py ${NSIM:-1000} 3 > gpurun_out/prof_plain_$TAG.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid -s 1 -c 1 \
     -o gpurun_out/prof_grid_$TAG python scripts/prof_grid.py ${NSIM:-1000} 3 > gpurun_out/ncu_$TAG.log 2>&1
  tail -2 gpurun_out/ncu_$TAG.log
fi
