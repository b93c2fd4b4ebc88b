"""One-row (closed-loop steady state) grid steps at N scenarios for ncu: the time-split
kernel by default, k_grid with argument 'no_ts'.  python scripts/prof_ts.py [n] [no_ts]"""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
ctx = _capi.context(0)
if "no_ts" in sys.argv:
    ctx.set_option("no_ts", 1)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
vp = 0.4
x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2])
for s in range(5):
    sc = _capi.make_scenarios(7 + s, 0, n, m.lo, m.span)
    res, _, _ = ctx.grid_step(prob, x0, vp, vp, 32, False, None, n, sc, False)
print("kernel", ctx.get_option("last_grid_kernel"), "row", res.row, "ms", res.kernel_ms)
if hasattr(ctx.lib, "rg_ts_timeline"):  # the instrumented build (EXTRA=-DRG_TS_TIMELINE)
    import ctypes
    tl = np.zeros((24, 64, 2), dtype=np.int64)  # kTsThreads / 32 warps
    ctx.lib.rg_ts_timeline(tl.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
    P0, P1, C0, C1 = 12, 13, 15, 16  # the chain warps after the 12 tanh warps
    base = tl[P0, 0, 0]
    nch = 32
    print("block 0 timeline, kcycles from P0's first chunk: T0 [go done] T1 | P0 [start arrive] "
          "| C0 [go done] | P1 | C1")
    for g in range(nch):
        f = lambda w: "%7.2f %7.2f" % ((tl[w, g, 0] - base) / 1e3, (tl[w, g, 1] - base) / 1e3)
        print("%2d  T0 %s  T1 %s | P0 %s | C0 %s | P1 %s | C1 %s" % (g, f(0), f(1), f(P0), f(C0),
                                                                     f(P1), f(C1)))
    per = lambda w, k: np.diff(tl[w, 4:nch, k]).mean()
    print("period per chunk (kcycles): T0 %.2f P0 %.2f C0 %.2f; busy per chunk: T0 %.2f P0 %.2f "
          "C0 %.2f" % (per(0, 1) / 1e3, per(P0, 1) / 1e3, per(C0, 1) / 1e3,
                       (tl[0, 4:nch, 1] - tl[0, 4:nch, 0]).mean() / 1e3,
                       (tl[P0, 4:nch, 1] - tl[P0, 4:nch, 0]).mean() / 1e3,
                       (tl[C0, 4:nch, 1] - tl[C0, 4:nch, 0]).mean() / 1e3))
