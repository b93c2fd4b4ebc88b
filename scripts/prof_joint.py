"""ncu driver: the persistent speculative joint search at 10k scenarios, the r = 2.5
transient from rest (kappa* = 0.5078; three candidates per round, one round)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2510_08288_b200 as rg  # noqa: E402
from paper_2510_08288_b200 import _capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = _capi.context(0)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
sc = _capi.make_scenarios(7 + 9000, 0, n, m.lo, m.span)
for s in range(reps):
    r = ctx.bisect_joint(prob, np.zeros(3), 0.0, 2.5, 8, None, n, sc)
    assert r.kappa == 0.5078125, r.kappa
    print(f"rep {s}: kernel {r.kernel_ms:.3f} ms")
