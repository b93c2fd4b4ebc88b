"""Golden C2 transient-binding variant: the real reference at N = 1000 scenarios.

SURVEY.md §8(d) C2, second variant (the style of the reference's acceptance criteria
3/4, tests/test_acceptance.py:88-146): state off equilibrium x0 = [tanh v_p, v_p,
tanh(v_p)/2] + U(+-0.05), v_p ~ U(-1, 1), request r ~ U(-2.5, 2.5), disturbances
scaled(0.02), j* = 256, M = 32, n_kappa = 8, 1000 scenarios, 16 trials.  For every
trial the unmodified reference computes
  * the grid step: fill_feasibility(backend="multicore") -> P (32 x 1000, stored packed),
    the stats dict, and extract_kappa_opt -> (kappa, v, feasible) as robust_rg_parallel
    applies it (governor.py:520-579);
  * Alg. 2: robust_rg_sequential -> (kappa, v, feasible, sims_run, early_terms)
    (governor.py:469-517).
The reference has no joint search; its kappa / feasible must equal Alg. 2's.
Writes tests/golden/c2_transient.npz.

Run in the build container (needs /root/reference):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_c2_transient_golden.py
"""

import time
from pathlib import Path

import numpy as np
from refgov import (ConstraintSet, DisturbanceModel, GovernorConfig, GovernorState,
                    extract_kappa_opt, fill_feasibility, grid_kappas, make_plant,
                    robust_rg_sequential, sample_scenarios, update_setpoint)

N, J_STAR, M, N_KAPPA, TRIALS, RANGE = 1000, 256, 32, 8, 16, 0.02

plant = make_plant("surrogate-fc")
box = ConstraintSet(-0.9, 0.9, anchor=0.0)
model = DisturbanceModel.scaled(RANGE, 3)
rng = np.random.default_rng(20261019)
rows = {k: [] for k in ("x0", "v_prev", "r", "seed", "p_packed", "grid", "stats", "seq")}
t0 = time.perf_counter()
for trial in range(TRIALS):
    v_p = float(rng.uniform(-1.0, 1.0))
    r = float(rng.uniform(-2.5, 2.5))
    x0 = np.array([np.tanh(v_p), v_p, np.tanh(v_p) / 2.0]) + rng.uniform(-0.05, 0.05, 3)
    seed = 31000 + trial
    scen = sample_scenarios(model, N, J_STAR + 1, seed=seed)
    stats = {}
    P = fill_feasibility("multicore", plant, x0, v_p, r, grid_kappas(M), scen, box, 0.05,
                         J_STAR, stats=stats)
    row, kappa = extract_kappa_opt(P)
    grid = [0.0, v_p, 0.0] if row is None else [kappa, update_setpoint(v_p, r, kappa), 1.0]
    cfg = GovernorConfig(j_star=J_STAR, n_sim=N, n_kappa=N_KAPPA, m_grid=M)
    seq = robust_rg_sequential(plant, x0, GovernorState(v_p), r, box, scen, cfg)
    rows["x0"].append(x0)
    rows["v_prev"].append(v_p)
    rows["r"].append(r)
    rows["seed"].append(seed)
    rows["p_packed"].append(np.packbits(P, axis=1))
    rows["grid"].append(grid)
    rows["stats"].append([stats["sims_run"], stats["early_terms"], stats["overflows"],
                          stats["ss_pruned_rows"], stats["dedup_rows"]])
    rows["seq"].append([seq.kappa_opt, seq.v_applied, float(seq.feasible),
                        seq.diagnostics["sims_run"], seq.diagnostics["early_terms"]])
out = {k: np.array(v) for k, v in rows.items()}
np.savez_compressed(Path(__file__).with_name("c2_transient.npz"), n_sim=N, j_star=J_STAR,
                    m_grid=M, n_kappa=N_KAPPA, range=RANGE, **out)
print(f"{TRIALS} trials in {time.perf_counter() - t0:.1f} s")
print("grid kappas", out["grid"][:, 0].tolist())
print("seq kappas", out["seq"][:, 0].tolist())
print("rows with violations per trial", [int((P_.sum(1) < N).sum()) for P_ in
                                         [np.unpackbits(p, axis=1)[:, :N] for p in out["p_packed"]]])
