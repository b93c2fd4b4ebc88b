import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
ctx = _capi.context(0)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
vp = 0.4
x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2])
spans = []
walls = []
for s in range(600):
    sc = _capi.make_scenarios(100 + s, 0, 10000, m.lo, m.span)
    t0 = time.perf_counter()
    res, _, _ = ctx.grid_step(prob, x0, vp, vp, 32, False, None, 10000, sc, False, timing=False, want_viol=False)
    walls.append(time.perf_counter() - t0)
    if s >= 100: spans.append(res.kernel_ms)
print("TS step at 10k: device span %.1f us, python-call wall %.1f us" % (np.median(spans)*1e3, np.median(walls[100:])*1e6))
