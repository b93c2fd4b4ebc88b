#!/bin/bash
# Round-2 profiles on one B200 (summaries only; .ncu-rep files dropped on the box):
# bench lines (C2 default, reference arm, C5, N=2 over gloo), the launch list of the
# default bench command, ncu --set full of k_grid (C2, 10k), k_joint_spec (10k transient)
# and k_grid_pairs (C5 regime).
TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c2.jsonl 2> gpurun_out/${TAG}_bench_c2.err
echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference_arm.jsonl 2>&1
echo "reference rc=$?"
timeout 900 python bench.py --workload c5 > gpurun_out/${TAG}_bench_c5.jsonl 2> gpurun_out/${TAG}_bench_c5.err
echo "c5 rc=$?"
RG_BENCH_DIST_BACKEND=gloo RG_BENCH_DEVICE=0 timeout 600 python bench.py --gpus 2 --steps 5 \
  --warmup 2 > gpurun_out/${TAG}_bench_n2_gloo.jsonl 2> gpurun_out/${TAG}_bench_n2_gloo.err
echo "n2 rc=$?"
SMALL="--steps 20 --warmup 3 --no-cpu-baseline --no-sweep --e2e-steps 5"
timeout 300 python bench.py $SMALL > gpurun_out/launch_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py $SMALL > gpurun_out/launch_ncu.log 2>&1
echo "launch list rc=$?"
prof() {  # name driver args kernel-regex cells workload
  local name=$1 drv=$2 args=$3 kre=$4 cells=$5 wl=$6
  python $drv $args > gpurun_out/prof_plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 \
     -o /tmp/prof_$name python $drv $args > gpurun_out/ncu_$name.log 2>&1
  echo "ncu $name rc=$?"
  python scripts/ncu_summary.py /tmp/prof_$name.ncu-rep $cells \
     gpurun_out/${TAG}_${name}_ncu.json "$wl" > /dev/null 2>&1
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > gpurun_out/${TAG}_${name}_ncu_raw.csv 2>/dev/null
  rm -f /tmp/prof_$name.ncu-rep
}
prof k_grid_1000 scripts/prof_grid.py "1000 3" "k_grid" $((32 * 1000 * 256)) \
  "k_grid: n_sim=1000, j*=256, M=32 (bench snapshot), staged SoA"
prof k_grid_10000 scripts/prof_grid.py "10000 3" "k_grid" $((32 * 10000 * 256)) \
  "k_grid: n_sim=10000, j*=256, M=32 (bench snapshot), staged SoA"
prof k_joint_spec_10000 scripts/prof_joint.py "10000 3" "k_joint_spec" $((3 * 10000 * 256)) \
  "k_joint_spec: n_sim=10000, r=2.5 transient, 3 candidates x 10k x 256 steps executed"
prof k_grid_pairs_512 scripts/prof_pairs.py "512 2" "k_grid_pairs" $((512 * 10000 * 256)) \
  "k_grid_pairs: 512 episodes x 10k scenarios, 1 live row each, fused RNG"
du -sh gpurun_out
