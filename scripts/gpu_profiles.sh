#!/bin/bash
# Round profiles on the box, keeping gpurun_out/ small: bench line (C2), reference arm,
# launch list, ncu --set full of k_grid at C2 (1000 scenarios) and at 10k, summarised
# on the box (scripts/ncu_summary.py + the raw page); the .ncu-rep files are dropped.
TAG=${TAG:-r}
mkdir -p gpurun_out
timeout 400 python bench.py --steps 1000 --warmup 10 --cpu-seconds 5 > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?"
timeout 400 python bench.py --impl reference --steps 200 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1
echo "reference rc=$?"
SMALL="--steps 20 --warmup 3 --no-cpu-baseline --no-sweep --e2e-steps 5"
timeout 300 python bench.py $SMALL > gpurun_out/launch_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py $SMALL > gpurun_out/launch_ncu.log 2>&1
echo "launch list rc=$?"
for N in 1000 10000; do
  python scripts/prof_grid.py $N 3 > gpurun_out/prof_plain_$N.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_grid -s 1 -c 1 \
     -o /tmp/prof_$N python scripts/prof_grid.py $N 3 > gpurun_out/ncu_$N.log 2>&1
  echo "ncu $N rc=$?"
  python scripts/ncu_summary.py /tmp/prof_$N.ncu-rep $((32 * N * 256)) \
     gpurun_out/${TAG}_k_grid_ncu_$N.json "n_sim=$N, j*=256, M=32 (bench snapshot), staged SoA" \
     > /dev/null 2>&1
  ncu -i /tmp/prof_$N.ncu-rep --page raw --csv > gpurun_out/${TAG}_k_grid_ncu_raw_$N.csv 2>/dev/null
  rm -f /tmp/prof_$N.ncu-rep
done
du -sh gpurun_out
