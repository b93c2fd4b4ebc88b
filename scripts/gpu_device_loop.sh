#!/bin/bash
# The device closed loop (k_loop_ts): parity (native loop tests, C3/C1 goldens), then C3 A/B
# (LIBS="name=path ..." variants beside the in-tree library; RG_NO_DEVICE_LOOP=1 = per-step loop).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_native_loop.py tests/test_gpu_parity.py -x -q \
  -p no:cacheprovider -k "native or device_loop or prelaunch or closed_loop" > gpurun_out/dl_tests.log 2>&1
echo "device-loop tests rc=$?" >> gpurun_out/dl_tests.log
tail -4 gpurun_out/dl_tests.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/dl_c3_$name.json 2> gpurun_out/dl_c3_$name.err
  python - gpurun_out/dl_c3_$name.json <<'PY'
import json, sys
f = sys.argv[1]
ls = [l for l in open(f).read().splitlines() if l.startswith("{")]
if not ls:
    print(f, "NO LINE", open(f.replace(".json", ".err")).read()[-800:]); sys.exit()
d = json.loads(ls[-1])
print(f, "ms/step %.5f" % d["ms_per_step"], "value %.4g" % d["value"], "launches", d.get("gpu_launches"), "device_loop", d.get("device_loop"))
PY
}
for i in 1 2; do
  run new_$i RG_X=1
  for L in ${LIBS}; do run ${L%%=*}_$i RG_LIB_PATH=${L#*=}; done
  run perstep_$i RG_NO_DEVICE_LOOP=1
done
