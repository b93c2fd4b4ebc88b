"""Per-step wall time of the native closed loop with and without pre-launched steps."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop

PLANT = rg.make_plant("surrogate-fc")
BOX = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
DESK = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
ctx = _capi.context(0)
for n in (1000, 10_000):
    cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=n)
    model = rg.DisturbanceModel.scaled(0.001, 3)
    for pre in (0, 1, 0, 1):
        ctx.set_option("no_prelaunch", 1 - pre)
        k0 = ctx.get_option("grid_step_kernels")
        t = time.perf_counter()
        rec = run_closed_loop(PLANT, BOX, model, cfg, DESK, 600, 7)
        dt = (time.perf_counter() - t) / 600 * 1e3
        k1 = ctx.get_option("grid_step_kernels")
        w = np.array([r[6] for r in rec.rows], dtype=float)
        print(f"n={n} pre={pre} ms/step={dt:.4f} kernels={k1-k0} wall_us p10/50/90/max="
              f"{np.percentile(w,10):.0f}/{np.percentile(w,50):.0f}/{np.percentile(w,90):.0f}/{w.max():.0f}"
              f" first10={w[:10].astype(int).tolist()} last_kernel={ctx.get_option('last_grid_kernel')}",
              flush=True)
ctx.set_option("no_prelaunch", 0)
