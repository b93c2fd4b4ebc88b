# Build the variants first, e.g. in paper_2510_08288_b200/csrc:
#   make -j4 EXTRA="-DRG_MW_MINB=7 -DRG_PAIRS_MINB=7" LIBDIR=../../scripts/micro/libs/mb7
# (RG_MW_MINB / RG_PAIRS_MINB were launch-bound macros of the probe build, not of the library.)
# Multi-wave k_grid (MOD form) and k_grid_pairs at 6 / 7 / 8 resident 64-thread blocks per SM
# (register caps 168 / 146 / 128): one library build per cap (scripts/micro/libs/mbN).
import os, subprocess, sys, json
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "micro")
ROOT = os.path.dirname(os.path.dirname(HERE))
CODE = r'''
import sys, time, json
sys.path.insert(0, %r)
import numpy as np, torch
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
ctx = _capi.context(0)
stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda", 0))
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
x0 = np.zeros(3); x0p = x0.ctypes.data
res = _capi.GridResult()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
out = {}
for n, reps in ((10000, 30), (100000, 8), (1 << 20, 3)):
    ts = []
    with torch.cuda.stream(stream):
        for s in range(reps + 1):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sc = _capi.make_scenarios(7 + s, 0, n, m.lo, m.span)
            _capi.check(ctx.lib.rg_grid_step(ctx.handle, prob, x0p, 0.0, 0.5, 32, 0, None, n, 0, sc, None, None, res, _capi.RG_ASYNC | _capi.RG_NO_TIMING))
            b.record(stream)
            torch.cuda.synchronize()
            if s: ts.append(a.elapsed_time(b))
    out["grid_%%d" %% n] = float(np.median(ts))
for E, rows in ((1024, 1), (128, 32)):
    vp = np.full(E, 0.4) if rows == 1 else np.zeros(E)
    r = np.full(E, 0.4) if rows == 1 else np.full(E, 0.5)
    X = np.stack([[np.tanh(v), v, np.tanh(v) / 2] for v in vp])
    ctx.grid_step_batch(prob, X, vp, r, list(range(E)), 0, 10000, m.lo, m.span, 32)
    t0 = time.perf_counter()
    for q in range(3):
        o = ctx.grid_step_batch(prob, X, vp, r, list(range(q*E, (q+1)*E)), 0, 10000, m.lo, m.span, 32)
    out["pairs_%%dx%%d" %% (E, rows)] = (time.perf_counter() - t0) / 3 * 1e3
    assert np.all(o[1] == 1.0)
print(json.dumps(out))
''' % ROOT
for mb in sys.argv[1:] or ["6", "7", "8"]:
    env = dict(os.environ, RG_LIB_PATH=os.path.join(HERE, "libs", "mb" + mb, "librefgov_b200.so"))
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print("mb" + mb, r.stdout.strip() or r.stderr[-800:], flush=True)
