#!/bin/bash
# ncu --set full of the C1 loop kernel and the one-row time-split step (after the split hash and
# the batch placement), summarised into gpurun_out/.
mkdir -p gpurun_out
timeout 200 python scripts/prof_c1.py > gpurun_out/prof_c1.log 2>&1; cat gpurun_out/prof_c1.log
cells=$(grep cell_steps gpurun_out/prof_c1.log | awk '{print $2}')
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_loop_bisect -c 1 \
  -o /tmp/prof_c1 python scripts/prof_c1.py > gpurun_out/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
python scripts/ncu_summary.py /tmp/prof_c1.ncu-rep $cells gpurun_out/k_loop_bisect_c1_ncu.json \
  "k_loop_bisect: the C1 desk trace (2000 steps, one scenario) in one launch"
bash scripts/gpu_prof_ts.sh
