"""Per-step device time of the closed loop on the device (k_loop_ts) at C3 and at 1k:
steps by live-row count, and the whole trace's wall clock per step."""
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
for n in (10_000, 1000):
    cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=n)
    model = rg.DisturbanceModel.scaled(0.001, 3)
    run_closed_loop(PLANT, BOX, model, cfg, DESK, 200, 3)
    for dl in (0, 1):
        ctx.set_option("no_device_loop", 1 - dl)
        t = time.perf_counter()
        rec = run_closed_loop(PLANT, BOX, model, cfg, DESK, 2000, 2024)
        wall = (time.perf_counter() - t) / 2000 * 1e6
        w = np.array([r[6] for r in rec.rows], dtype=float)
        sims = np.array([int(d.split(",")[4]) for d in rec.diag_rows])
        rows = sims // n
        msg = f"n={n} device_loop={dl} wall/step {wall:.1f} us; step wall_us sum/step {w.sum()/2000:.1f}"
        for k in sorted(set(rows.tolist()))[:6]:
            sel = rows == k
            msg += f" | {k} rows: {sel.sum()} steps, median {np.median(w[sel]):.0f} us"
        print(msg, flush=True)
ctx.set_option("no_device_loop", 0)
