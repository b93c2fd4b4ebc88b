"""Chunk timeline of the last block (one unit at 1k scenarios): the standalone time-split
step vs a step inside the device closed loop.  Needs the RG_TS_TIMELINE build with
RG_TS_TL_BLOCK=(gridDim.x-1) via RG_LIB_PATH."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
from paper_2510_08288_b200.harness import run_closed_loop

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
ctx = _capi.context(0)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)


def show(tag):
    tl = np.zeros((24, 64, 2), dtype=np.int64)
    ctx.lib.rg_ts_timeline(tl.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
    P0, C0 = 12, 15
    base = tl[P0, 0, 0]
    per = np.diff(tl[C0, 4:32, 1]).mean() / 1e3
    print(f"{tag}: C0 last chunk done {(tl[C0, 31, 1] - base) / 1e3:.2f} kcycles after P0's first; "
          f"period C0 {per:.2f}, P0 {np.diff(tl[P0, 4:32, 1]).mean() / 1e3:.2f}, "
          f"T0 busy {(tl[0, 4:32, 1] - tl[0, 4:32, 0]).mean() / 1e3:.2f}, P0 busy "
          f"{(tl[P0, 4:32, 1] - tl[P0, 4:32, 0]).mean() / 1e3:.2f}", flush=True)


vp = 0.4
x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2])
for s in range(5):
    sc = _capi.make_scenarios(7 + s, 0, n, m.lo, m.span)
    ctx.grid_step(prob, x0, vp, vp, 32, False, None, n, sc, False)
show(f"standalone k_grid_ts n={n}")
cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=n)
run_closed_loop(rg.make_plant("surrogate-fc"), rg.ConstraintSet(-0.9, 0.9, anchor=0.0), m, cfg,
                [0.4] * 60, 60, 3, x0=x0, v0=vp)
show(f"k_loop_ts step 59 n={n}")
