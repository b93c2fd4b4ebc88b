#!/bin/bash
# The device closed loop (k_loop_ts): parity (native loop tests, C3/C1 goldens), then C3 A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_native_loop.py tests/test_gpu_parity.py -x -q \
  -p no:cacheprovider -k "native or device_loop or prelaunch or closed_loop" > gpurun_out/dl_tests.log 2>&1
echo "device-loop tests rc=$?" >> gpurun_out/dl_tests.log
tail -4 gpurun_out/dl_tests.log
for i in 1 2; do
  timeout 300 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/dl_c3_on_$i.json 2> gpurun_out/dl_c3_on_$i.err
  RG_NO_DEVICE_LOOP=1 timeout 300 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/dl_c3_off_$i.json 2> gpurun_out/dl_c3_off_$i.err
done
for f in gpurun_out/dl_c3_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
ls = [l for l in open(f).read().splitlines() if l.startswith("{")]
if not ls:
    print(f, "NO LINE", open(f.replace(".json", ".err")).read()[-800:]); sys.exit()
d = json.loads(ls[-1])
print(f, "ms/step", d["ms_per_step"], "value %.4g" % d["value"], "launches", d.get("gpu_launches"), "frac", (d.get("roofline") or {}).get("frac"))
PY
done
