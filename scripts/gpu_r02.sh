#!/bin/bash
# Round-2 development pass on one B200: tests + smoke, the default bench line, the
# reference arm, the N=2 path over gloo on one GPU, and a reduced C5 run.
mkdir -p gpurun_out
PYTEST_TIMEOUT=900 bash scripts/gpu_tests.sh
timeout 600 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err
echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
echo "ref rc=$?"
RG_BENCH_DIST_BACKEND=gloo RG_BENCH_DEVICE=0 timeout 600 python bench.py --gpus 2 --steps 5 \
  --warmup 2 > gpurun_out/bench_n2_gloo.log 2> gpurun_out/bench_n2_gloo.err
echo "n2 rc=$?"
timeout 900 python bench.py --workload c5 ${C5_ARGS:---episodes 512 --steps 3 --warmup 2} \
  > gpurun_out/bench_c5.log 2> gpurun_out/bench_c5.err
echo "c5 rc=$?"
for f in bench_default bench_ref bench_n2_gloo bench_c5; do
  echo "== $f"; tail -c 1500 gpurun_out/$f.log; tail -3 gpurun_out/$f.err; done
