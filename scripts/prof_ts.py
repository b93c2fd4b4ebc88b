"""One-row (closed-loop steady state) grid steps at N scenarios for ncu: the time-split
kernel by default, k_grid with argument 'no_ts'.  python scripts/prof_ts.py [n] [no_ts]"""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
ctx = _capi.context(0)
if "no_ts" in sys.argv:
    ctx.set_option("no_ts", 1)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
vp = 0.4
x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2])
for s in range(5):
    sc = _capi.make_scenarios(7 + s, 0, n, m.lo, m.span)
    res, _, _ = ctx.grid_step(prob, x0, vp, vp, 32, False, None, n, sc, False)
print("kernel", ctx.get_option("last_grid_kernel"), "row", res.row, "ms", res.kernel_ms)
