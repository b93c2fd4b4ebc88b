#!/bin/bash
# ncu --set full of the device closed loop (k_loop_ts, 200 steps at 10k), summarised.
mkdir -p gpurun_out
timeout 200 python scripts/prof_loop.py > gpurun_out/prof_loop.log 2>&1; cat gpurun_out/prof_loop.log
cells=$(grep cell_steps gpurun_out/prof_loop.log | awk '{print $2}')
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_loop_ts -c 1 \
  -o /tmp/prof_loop python scripts/prof_loop.py > gpurun_out/ncu_loop.log 2>&1
echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/prof_loop.ncu-rep $cells gpurun_out/k_loop_ts_10000_ncu.json \
  "k_loop_ts: 200-step desk closed loop at 10k scenarios in one launch (fused RNG)"
ncu -i /tmp/prof_loop.ncu-rep --page raw --csv > gpurun_out/k_loop_ts_10000_ncu_raw.csv
