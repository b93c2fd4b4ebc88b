# Ran once in round 2 against the ROUND-1 library (git 23d38c9, which still had the lanes-per-cell
# forms), built to scripts/micro/oldlib with its package copied to scripts/micro/oldpkg (both
# git-ignored).  Output: profiles/r02_lpc_probe_round1_library.txt.
# Round-1 library (lanes-per-cell forms) on the latency-bound shapes: 10k scenarios with ONE
# live row (a closed-loop step: v_prev == r) and Alg. 2 at 10k (r = 2.5 transient).
import os, sys, time
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "micro")
os.environ["RG_LIB_PATH"] = os.path.join(HERE, "oldlib", "librefgov_b200.so")
sys.path.insert(0, os.path.join(HERE, "oldpkg"))
import numpy as np
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
ctx = _capi.context(0)
m = rg.DisturbanceModel.scaled(0.001, 3)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
for n in (3000, 10000, 30000):
    sc = _capi.make_scenarios(7, 0, n, m.lo, m.span)
    x0 = np.array([np.tanh(0.4), 0.4, np.tanh(0.4) / 2])
    for lpc in (1, 2, 4):
        for rng_mode in ("staged", "fused"):
            f = lambda: ctx.grid_step(prob, x0, 0.4, 0.4, 32, False, None, n, sc, False, abandon=True, rng_mode=rng_mode, lpc=lpc, timing=True, want_viol=False)
            f()
            ts = []
            for _ in range(20):
                r = f()[0]
                ts.append(r.kernel_ms)
            print(f"grid 1-row n={n} lpc={lpc} {rng_mode}: {np.median(ts):.4f} ms row={r.row}")
    x0 = np.zeros(3)
    for lpc in (1, 2, 4):
        f = lambda: ctx.bisect(prob, x0, 0.0, 2.5, 8, None, n, sc, lpc=lpc)[0]
        f(); ts = []
        for _ in range(20):
            r = f(); ts.append(r.kernel_ms)
        print(f"alg2 n={n} lpc={lpc}: {np.median(ts):.4f} ms kappa={r.kappa}")
