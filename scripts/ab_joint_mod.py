"""A/B: the persistent joint search with and without the operand-modifier tanh forms
(rg_set_option "joint_mod"), r = 2.5 transient and a C2-snapshot search, event times."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
ctx = _capi.context(0)
m = rg.DisturbanceModel.scaled(0.001, 3)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
for n in (1000, 3000, 10_000, 30_000):
    sc = _capi.make_scenarios(7 + 9000, 0, n, m.lo, m.span)
    for r in (2.5, 0.5):
        out = {}
        for mod in (0, 1, 0, 1):
            ctx.set_option("joint_mod", mod)
            ctx.bisect_joint(prob, np.zeros(3), 0.0, r, 8, None, n, sc)
            ts = [ctx.bisect_joint(prob, np.zeros(3), 0.0, r, 8, None, n, sc).kernel_ms
                  for _ in range(15)]
            out.setdefault(mod, []).append(float(np.median(ts)))
        print(f"n={n} r={r}: mod0 {min(out[0]):.4f} ms  mod1 {min(out[1]):.4f} ms")
