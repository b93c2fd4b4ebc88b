"""A/B of two library builds on the C2 step (event time of L2-flushed steps and the k_grid
device span), alternated.  A = scripts/micro/abA (+ its package copy in scripts/micro/abApkg),
B = the tree's own build."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CODE = r'''
import sys, json
sys.path.insert(0, "__PKG__")
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
ts = []
with torch.cuda.stream(stream):
    for s in range(820):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sc = _capi.make_scenarios(7 + s, 0, 1000, m.lo, m.span)
        _capi.check(ctx.lib.rg_grid_step(ctx.handle, prob, x0p, 0.0, 0.5, 32, 0, None, 1000, 0,
                                         sc, None, None, res, _capi.RG_ASYNC | _capi.RG_NO_TIMING))
        b.record(stream)
        if s >= 20:
            ts.append((a, b))
        if s % 50 == 49:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
ev = [x.elapsed_time(y) for x, y in ts]
sync = _capi.GridResult()
spans = []
for s in range(220):
    sc = _capi.make_scenarios(20000 + s, 0, 1000, m.lo, m.span)
    _capi.check(ctx.lib.rg_grid_step(ctx.handle, prob, x0p, 0.0, 0.5, 32, 0, None, 1000, 0, sc,
                                     None, None, sync, _capi.RG_NO_TIMING))
    if s >= 20:
        spans.append(sync.kernel_ms * 1e3)
print(json.dumps({"event_ms_median": float(np.median(ev)), "event_ms_mean": float(np.mean(ev)),
                  "span_us": float(np.median(spans))}))
'''


def run(tag, pkg, lib):
    env = dict(os.environ, RG_LIB_PATH=lib)
    r = subprocess.run([sys.executable, "-c", CODE.replace("__PKG__", pkg)], env=env,
                       capture_output=True, text=True)
    print(tag, r.stdout.strip()[-300:] or r.stderr[-800:], flush=True)


A = (os.path.join(HERE, "micro", "abApkg"), os.path.join(HERE, "micro", "abA", "librefgov_b200.so"))
B = (ROOT, os.path.join(ROOT, "paper_2510_08288_b200", "_lib", "librefgov_b200.so"))
for rep in range(3):
    run("A", *A)
    run("B", *B)
