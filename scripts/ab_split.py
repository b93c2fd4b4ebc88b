"""One-row (steady closed-loop) grid steps through the C ABI at several scenario counts:
mean host wall time per call over 400 calls (the time-split kernel with the fused RNG)."""
import sys, time
import numpy as np
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
for n in (1000, 2000, 4000, 4700, 10000):
    scs = [_capi.make_scenarios(7 + s, 0, n, m.lo, m.span) for s in range(400)]
    for sc in scs[:20]:
        ctx.grid_step(prob, x0, vp, vp, 32, False, None, n, sc, False)
    t0 = time.perf_counter()
    for sc in scs:
        res, _, _ = ctx.grid_step(prob, x0, vp, vp, 32, False, None, n, sc, False)
    dt = (time.perf_counter() - t0) / len(scs) * 1e6
    print(f"n={n}: {dt:.1f} us per one-row step (kernel {ctx.get_option('last_grid_kernel')})",
          flush=True)
