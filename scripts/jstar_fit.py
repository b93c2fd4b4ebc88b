"""k_grid time vs horizon at fixed scenario count: fixed overhead + per-step slope."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2510_08288_b200 as rg  # noqa: E402
from paper_2510_08288_b200 import _capi  # noqa: E402

n_sim = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
ctx = _capi.context(0)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
m = rg.DisturbanceModel.scaled(0.001, 3)
rows = []
for J in (1, 2, 8, 32, 64, 128, 256, 512):
    prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, J, 0)
    ts, tk = [], []
    for s in range(60):
        scen = _capi.make_scenarios(7 + s, 0, n_sim, m.lo, m.span)
        res, _, _ = ctx.grid_step(prob, np.zeros(3), 0.0, 0.5, 32, False, None, n_sim, scen,
                                  False)
        if s >= 10:
            ts.append(res.kernel_ms * 1e3)
        res2, _, _ = ctx.grid_step(prob, np.zeros(3), 0.0, 0.5, 32, False, None, n_sim, scen,
                                   False, timing=False)
        if s >= 10:
            tk.append(res2.kernel_ms * 1e3)
    rows.append((J, np.median(ts), np.median(tk)))
    print(f"J={J:4d}  events {np.median(ts):8.1f} us   globaltimer {np.median(tk):8.1f} us")
J = np.array([r[0] for r in rows], float)
t = np.array([r[1] for r in rows])
A = np.vstack([np.ones_like(J), J]).T
c, *_ = np.linalg.lstsq(A[J >= 32], t[J >= 32], rcond=None)
print(f"fit (J>=32): {c[0]:.1f} us fixed + {c[1]:.4f} us/step ({c[1]*1e-6*1.965e9:.0f} cycles/step)")
