"""The persistent joint search with its kappa = 1 probe on the time-split kernel vs inside
the search: steady state (r = v_prev) and the r = 2.5 transient, 1k and 10k scenarios,
wall time of the C-ABI call (sync), median of 200."""
import sys
import time
import numpy as np
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi

ctx = _capi.context(0)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
for n in (1000, 10_000):
    for name, vp, r in (("steady r=v_prev=0.4", 0.4, 0.4), ("transient 0 -> 2.5", 0.0, 2.5)):
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2])
        line = [f"n={n} {name}:"]
        for probe in (0, 1, 0, 1):
            ctx.set_option("no_ts_probe", 0 if probe else 1)
            ts = []
            for s in range(220):
                sc = _capi.make_scenarios(9 + s, 0, n, m.lo, m.span)
                t0 = time.perf_counter()
                j = ctx.bisect_joint(prob, x0, vp, r, 8, None, n, sc)
                if s >= 20:
                    ts.append(time.perf_counter() - t0)
            line.append(f"{'ts-probe' if probe else 'inline'} {np.median(ts) * 1e3:.4f} ms"
                        f" (kappa {j.kappa}, cells {j.cells})")
        print("  ".join(line), flush=True)
ctx.set_option("no_ts_probe", 0)
