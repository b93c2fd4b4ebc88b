#!/bin/bash
mkdir -p gpurun_out
python scripts/prof_ts.py 10000
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_grid_ts -s 2 -c 1 \
  -o gpurun_out/k_grid_ts_10000 python scripts/prof_ts.py 10000 > gpurun_out/ncu_ts.log 2>&1
echo "ncu rc=$?"
