#!/bin/bash
# ncu --set full of the time-split grid step (one-row closed-loop step, 10k and 1k scenarios),
# summarised into gpurun_out/ (scripts/ncu_summary.py) plus the raw page.
mkdir -p gpurun_out
for n in 10000 1000; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_grid_ts -s 2 -c 1 \
    -o /tmp/prof_ts_$n python scripts/prof_ts.py $n > gpurun_out/ncu_ts_$n.log 2>&1
  echo "ncu $n rc=$?"
  python scripts/ncu_summary.py /tmp/prof_ts_$n.ncu-rep $((n * 256)) \
    gpurun_out/k_grid_ts_${n}_ncu.json "k_grid_ts: one live row, n_sim=$n, j*=256, fused RNG"
  ncu -i /tmp/prof_ts_$n.ncu-rep --page raw --csv > gpurun_out/k_grid_ts_${n}_ncu_raw.csv
done
