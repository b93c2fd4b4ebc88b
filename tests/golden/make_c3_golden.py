"""Golden C3 prefix: the real reference's desk-scale closed loop at n_sim = 10,000.

BASELINE.json configs[2] (10k scenarios, the desk-scale setpoint trace) run by the
unmodified reference (`refgov.run_closed_loop`, `harness.py:138-224`, multicore
fill) for all 2000 steps of the desk-scale profile (STEPS env var to truncate): the rise
from rest to r = 0.4, the r = 2.5 step at t = 400, r = -2.5 at t = 1000 and r = 0.2
at t = 1600.  Writes tests/golden/c3_10k_trace.npz with the rows
(v_t, y_t, kappa_t, feasible_t) per step.

Run in the build container (needs /root/reference):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_c3_golden.py
"""

import os
from pathlib import Path

import numpy as np
from refgov import load_config, run_closed_loop

STEPS = int(os.environ.get("STEPS", "2000"))

setup = load_config({"governor": {"n_sim": 10000, "backend": "multicore"}})
rec = run_closed_loop(setup.plant, setup.cset, setup.model, setup.governor, setup.profile,
                      STEPS, setup.seed)
assert not rec.aborted
trace = np.array([[row[2], row[3], row[4], float(row[5])] for row in rec.rows])
np.savez_compressed(Path(__file__).with_name("c3_10k_trace.npz"), trace=trace,
                    n_sim=10000, steps=STEPS, seed=setup.seed)
print(f"wrote {len(trace)} steps; kappa range {trace[:, 2].min()}..{trace[:, 2].max()}")
