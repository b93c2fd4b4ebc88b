"""Golden C4 step: the real reference's robust grid step at 2^20 scenarios, j* = 256.

BASELINE.json configs[3] at its full per-step size, run by the unmodified reference
(`refgov.fill_feasibility(backend="multicore")`, `governor.py:245-348`, then
`extract_kappa_opt`, `governor.py:351-377`) on a transient-binding snapshot
(scaled(0.02) disturbances, state off equilibrium, a large setpoint request), so
that some candidate rows fail on some scenarios and others hold on all 2^20.
The 32 x 2^20 matrix P is stored as its per-row feasible counts and the sha256
of its packed bits; the step's (kappa, v, feasible) are stored as doubles.
Writes tests/golden/c4_1m_step.npz.

Run in the build container (needs /root/reference, ~7 GB of RAM):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_c4_golden.py
"""

import hashlib
import time
from pathlib import Path

import numpy as np
from refgov import (ConstraintSet, DisturbanceModel, extract_kappa_opt, fill_feasibility,
                    grid_kappas, make_plant, sample_scenarios, update_setpoint)

N, J_STAR, M, SEED = 1 << 20, 256, 32, 20261019
V_PREV, R = 0.2, 2.4
X0 = np.array([np.tanh(V_PREV), V_PREV, np.tanh(V_PREV) / 2.0]) + 0.03
RANGE = 0.02

plant = make_plant("surrogate-fc")
box = ConstraintSet(-0.9, 0.9, anchor=0.0)
t0 = time.perf_counter()
scen = sample_scenarios(DisturbanceModel.scaled(RANGE, 3), N, J_STAR + 1, seed=SEED)
t1 = time.perf_counter()
P = fill_feasibility("multicore", plant, X0, V_PREV, R, grid_kappas(M), scen, box, 0.05, J_STAR)
t2 = time.perf_counter()
row, kappa = extract_kappa_opt(P)
if row is None:
    result = np.array([0.0, V_PREV, 0.0])
else:
    result = np.array([kappa, update_setpoint(V_PREV, R, kappa), 1.0])
np.savez_compressed(
    Path(__file__).with_name("c4_1m_step.npz"),
    n_sim=N, j_star=J_STAR, m_grid=M, seed=SEED, v_prev=V_PREV, r=R, x0=X0, range=RANGE,
    row_counts=P.sum(axis=1).astype(np.int64),
    p_sha=np.frombuffer(hashlib.sha256(np.packbits(P, axis=1).tobytes()).digest(), np.uint8),
    result=result)
print(f"sample {t1 - t0:.1f} s, fill {t2 - t1:.1f} s; row counts {P.sum(axis=1).tolist()}; "
      f"result {result.tolist()}")
