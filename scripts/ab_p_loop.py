"""A caller's own closed-loop step through robust_rg_parallel with P returned (the default
keep_matrix=True) in steady state (r = v_prev: one live row) at 1k and 10k scenarios: the
host row plan (time-split kernel) against device-derived rows (k_grid), wall time per call."""
import sys
import time
import numpy as np
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi

plant = rg.make_plant("surrogate-fc")
box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
model = rg.DisturbanceModel.scaled(0.001, 3)
ctx = _capi.context(0)
vp = 0.4
x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2])
for n in (1000, 10_000):
    cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=n)
    for rep in range(2):
        for plan in (1, 0):
            ctx.set_option("no_row_plan", 0 if plan else 1)
            for s in range(20):
                rg.robust_rg_parallel(plant, x0, rg.GovernorState(vp), vp, box,
                                      rg.sample_scenarios(model, n, 257, seed=s), cfg)
            t0 = time.perf_counter()
            for s in range(300):
                res = rg.robust_rg_parallel(plant, x0, rg.GovernorState(vp), vp, box,
                                            rg.sample_scenarios(model, n, 257, seed=100 + s), cfg)
            dt = (time.perf_counter() - t0) / 300 * 1e3
            print(f"n={n} row plan={plan}: {dt:.4f} ms per call (P {res.matrix.shape}, kernel "
                  f"{ctx.get_option('last_grid_kernel')})", flush=True)
ctx.set_option("no_row_plan", 0)
