"""Golden Alg. 2 step at 2^20 scenarios: the real reference's robust_rg_sequential.

Same snapshot and scenarios as make_c4_golden.py (BASELINE.json configs[3]), run by
the unmodified reference (`refgov.robust_rg_sequential`, `governor.py:469-517`:
one `_bisect_kappa` per scenario, kappa_opt = min, feasible = AND).  Stores
(kappa, v, feasible, sims_run, early_terms).  Writes tests/golden/c4_1m_seq.npz.

Run in the build container (needs /root/reference, ~7 GB of RAM, a few minutes):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_c4_seq_golden.py
"""

import time
from pathlib import Path

import numpy as np
from refgov import (ConstraintSet, DisturbanceModel, GovernorConfig, GovernorState, make_plant,
                    robust_rg_sequential, sample_scenarios)

with np.load(Path(__file__).with_name("c4_1m_step.npz")) as z:
    g = {k: z[k] for k in z.files}
n, j_star = int(g["n_sim"]), int(g["j_star"])
scen = sample_scenarios(DisturbanceModel.scaled(float(g["range"]), 3), n, j_star + 1,
                        seed=int(g["seed"]))
t0 = time.perf_counter()
res = robust_rg_sequential(make_plant("surrogate-fc"), g["x0"], GovernorState(float(g["v_prev"])),
                           float(g["r"]), ConstraintSet(-0.9, 0.9, anchor=0.0), scen,
                           GovernorConfig(j_star=j_star, n_sim=n, n_kappa=8))
dt = time.perf_counter() - t0
d = res.diagnostics
out = np.array([res.kappa_opt, res.v_applied, float(res.feasible), d["sims_run"],
                d["early_terms"]])
np.savez_compressed(Path(__file__).with_name("c4_1m_seq.npz"), result=out, seconds=dt)
print(f"robust_rg_sequential at n={n}: {dt:.1f} s, result {out.tolist()}")
