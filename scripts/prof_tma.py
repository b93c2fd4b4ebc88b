"""A few C2 steps with the TMA-fed ring (tma_ring) for ncu."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
ctx = _capi.context(0)
ctx.set_option("tma_ring", 1)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
for s in range(4):
    sc = _capi.make_scenarios(7 + s, 0, 1000, m.lo, m.span)
    res, _, _ = ctx.grid_step(prob, np.zeros(3), 0.0, 0.5, 32, False, None, 1000, sc, False)
print(res.row, res.kernel_ms)
