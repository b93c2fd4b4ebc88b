"""Golden closed loops with transients: the real reference's run_closed_loop (harness.py:138-224,
multicore fill) on two configurations where several candidate rows are live at once, so the
device loop's steps need several time-split passes and the gate / dedup / prefix paths work:

  lit:    n_sim 2000, j* 256, M 32, literal Eq. 4, disturbances scaled(0.02), references jumping
          0.4 -> 2.5 -> -2.5 -> 1.0 -> -1.0 every 60 steps, 300 steps, seed 77;
  prefix: n_sim 1500, j* 128, M 16, prefix mode, scaled(0.01), the same jumps, 300 steps, seed 5.

Writes tests/golden/loop_transient.npz with the rows (v_t, y_t, kappa_t, feasible_t) and the
diagnostics (sims_run, early_terms) per step.  Run in the build container (needs /root/reference):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \\
        python tests/golden/make_loop_transient_golden.py
"""

from pathlib import Path

import numpy as np
from refgov import (ConstraintSet, DisturbanceModel, GovernorConfig, ReferenceProfile,
                    make_plant, run_closed_loop)

PROFILE = ((0, 0.4), (60, 2.5), (120, -2.5), (180, 1.0), (240, -1.0))
CASES = {
    "lit": dict(n_sim=2000, j_star=256, m_grid=32, prefix_mode=False, scale=0.02, seed=77),
    "prefix": dict(n_sim=1500, j_star=128, m_grid=16, prefix_mode=True, scale=0.01, seed=5),
}
STEPS = 300

out = {"steps": STEPS, "profile": np.array(PROFILE, dtype=float)}
plant = make_plant("surrogate-fc")
box = ConstraintSet(-0.9, 0.9, anchor=0.0)
for name, c in CASES.items():
    cfg = GovernorConfig(j_star=c["j_star"], m_grid=c["m_grid"], n_sim=c["n_sim"],
                         prefix_mode=c["prefix_mode"], backend="multicore")
    rec = run_closed_loop(plant, box, DisturbanceModel.scaled(c["scale"], 3), cfg,
                          ReferenceProfile(PROFILE), STEPS, c["seed"])
    assert not rec.aborted, rec.abort_reason
    out[f"{name}_trace"] = np.array([[r[2], r[3], r[4], float(r[5])] for r in rec.rows])
    out[f"{name}_diag"] = np.array([[int(d.split(",")[4]), int(d.split(",")[5])]
                                    for d in rec.diag_rows], dtype=np.int64)
    for k, v in c.items():
        out[f"{name}_{k}"] = v
    sims = out[f"{name}_diag"][:, 0]
    print(f"{name}: {len(rec.rows)} steps; live rows per step max {sims.max() // c['n_sim']}, "
          f"mean {sims.mean() / c['n_sim']:.2f}")
np.savez_compressed(Path(__file__).with_name("loop_transient.npz"), **out)
