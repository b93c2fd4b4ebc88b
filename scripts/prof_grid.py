"""Small driver for ncu: a few fused grid steps at the bench workload (C2, N=1000)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2510_08288_b200 as rg  # noqa: E402
from paper_2510_08288_b200 import _capi  # noqa: E402

n_sim = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = _capi.context(0)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
for s in range(steps):
    scen = _capi.make_scenarios(7 + s, 0, n_sim, m.lo, m.span)
    res, viol, _ = ctx.grid_step(prob, np.zeros(3), 0.0, 0.5, 32, False, None, n_sim, scen, False)
    assert res.row == 31, res.row
    print(f"step {s}: kernel {res.kernel_ms:.3f} ms")
