"""Device time of the three robust searches at N scenarios (transient step r=2.5 from rest,
kappa* ~ 0.5: every bisection runs all n_kappa + 1 candidates)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2510_08288_b200 as rg  # noqa: E402
from paper_2510_08288_b200 import _capi  # noqa: E402

ctx = _capi.context(0)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
x0 = np.zeros(3)
for n in [int(a) for a in (sys.argv[1:] or ["1000", "10000", "100000", "1000000"])]:
    sc = _capi.make_scenarios(7, 0, n, m.lo, m.span)
    out = {}
    for name, fn in (("grid", lambda: ctx.grid_step(prob, x0, 0.0, 2.5, 32, False, None, n, sc,
                                                     False, abandon=True)[0]),
                     ("alg2", lambda: ctx.bisect(prob, x0, 0.0, 2.5, 8, None, n, sc)[0]),
                     ("joint", lambda: ctx.bisect_joint(prob, x0, 0.0, 2.5, 8, None, n, sc))):
        fn()
        reps = 5 if n >= 100000 else 20
        t0 = time.perf_counter()
        for _ in range(reps):
            r = fn()
        wall = (time.perf_counter() - t0) / reps * 1e3
        k = (r.row / 31 if name == "grid" else r.kappa)
        out[name] = (wall, k)
    print(f"N={n:8d} " + "  ".join(f"{k}: {w:8.3f} ms (kappa {kk:.6f})" for k, (w, kk)
                                    in out.items()), flush=True)
