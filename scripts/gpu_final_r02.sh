#!/bin/bash
# Round-2 closing pass on one B200: tests + smoke, then every bench line this round reports
# (C2 default, reference arm, C3, C4 through the NCCL path at one rank, C5, the N=2 path over
# gloo), into gpurun_out/final_*.jsonl.
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
timeout 600 python bench.py > gpurun_out/final_c2.jsonl 2> gpurun_out/final_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/final_c2_reference.jsonl 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --workload c3 > gpurun_out/final_c3.jsonl 2>&1; echo "c3 rc=$?"
timeout 600 python bench.py --impl reference --workload c3 > gpurun_out/final_c3_reference.jsonl 2>&1; echo "c3 ref rc=$?"
RG_BENCH_FORCE_DIST=1 timeout 600 python bench.py --workload c4 > gpurun_out/final_c4_world1.jsonl 2>&1; echo "c4 rc=$?"
timeout 900 python bench.py --workload c5 > gpurun_out/final_c5.jsonl 2>&1; echo "c5 rc=$?"
RG_BENCH_DIST_BACKEND=gloo RG_BENCH_DEVICE=0 timeout 600 python bench.py --gpus 2 --steps 5 \
  --warmup 2 > gpurun_out/final_n2_gloo.jsonl 2>&1; echo "n2 rc=$?"
for f in gpurun_out/final_*.jsonl; do
  python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
ls = [l for l in open(f).read().splitlines() if l.startswith("{")]
if not ls:
    print(f, "NO LINE"); sys.exit()
d = json.loads(ls[-1])
print(f, "value %.4g" % (d.get("value") or 0), "ms/step", d.get("ms_per_step"),
      "e2e", (d.get("e2e") or {}).get("ms_per_step"), "frac", (d.get("roofline") or {}).get("frac"))
PY
done
timeout 300 python bench.py --workload c1 > gpurun_out/final_c1.jsonl 2>&1; echo "c1 rc=$?"
timeout 300 python bench.py --impl reference --workload c1 > gpurun_out/final_c1_reference.jsonl 2>&1; echo "c1 ref rc=$?"
for f in gpurun_out/final_c1*.jsonl; do
  python -c "
import json; d=json.loads([l for l in open('$f') if l.startswith('{')][-1]); print('$f', 'ms/step', d.get('ms_per_step'))"
done
