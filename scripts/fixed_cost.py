"""Fixed cost of the C2 grid step: events around rg_grid_step at short horizons,
staged (k_gen_soa + k_grid, PDL) vs fused RNG (k_grid alone)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2510_08288_b200 as rg  # noqa: E402
from paper_2510_08288_b200 import _capi  # noqa: E402

ctx = _capi.context(0)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
m = rg.DisturbanceModel.scaled(0.001, 3)
for J in (1, 4, 16, 256):
    prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, J, 0)
    for mode in ("staged", "fused"):
        ev, gt = [], []
        for s in range(80):
            scen = _capi.make_scenarios(7 + s, 0, 1000, m.lo, m.span)
            res, _, _ = ctx.grid_step(prob, np.zeros(3), 0.0, 0.5, 32, False, None, 1000, scen,
                                      False, rng_mode=mode)
            res2, _, _ = ctx.grid_step(prob, np.zeros(3), 0.0, 0.5, 32, False, None, 1000, scen,
                                       False, rng_mode=mode, timing=False)
            if s >= 20:
                ev.append(res.kernel_ms * 1e3)
                gt.append(res2.kernel_ms * 1e3)
        print(f"J={J:4d} {mode:7s} events {np.median(ev):7.1f} us  k_grid span {np.median(gt):7.1f} us",
              flush=True)
