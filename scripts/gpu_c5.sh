#!/bin/bash
# C5 on one B200: the full 4096 x 10k batch (5 timed closed-loop steps after 3), and the
# fused / staged crossover of the batched step at 1 and 3 live rows per episode.
mkdir -p gpurun_out
timeout 900 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/bench_c5_full.log 2> gpurun_out/bench_c5_full.err
echo "c5 rc=$?"; tail -c 1200 gpurun_out/bench_c5_full.log; tail -3 gpurun_out/bench_c5_full.err
timeout 600 python - <<'PY' > gpurun_out/c5_modes.log 2>&1
import time, numpy as np, sys
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
ctx = _capi.context(0)
m = rg.DisturbanceModel.scaled(0.001, 3)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9, 0.0), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
for E, rows in ((1024, 1), (1024, 3), (256, 32)):
    vp = np.full(E, 0.4)
    r = np.full(E, 0.4) if rows == 1 else (np.full(E, 0.45) if rows == 3 else np.full(E, 0.5))
    if rows == 32: vp = np.zeros(E)
    X = np.stack([[np.tanh(v), v, np.tanh(v) / 2] for v in vp])
    seeds = list(range(E))
    for mode in ("fused", "staged"):
        kw = {mode: True}
        ctx.grid_step_batch(prob, X, vp, r, seeds, 0, 10000, m.lo, m.span, 32, **kw)
        t0 = time.perf_counter()
        for rep in range(3):
            out = ctx.grid_step_batch(prob, X, vp, r, seeds, 0, 10000, m.lo, m.span, 32, **kw)
        dt = (time.perf_counter() - t0) / 3
        print(E, "episodes", rows, "rows requested", mode, round(dt * 1e3, 2), "ms", "kappa0", out[1][0])
PY
cat gpurun_out/c5_modes.log
