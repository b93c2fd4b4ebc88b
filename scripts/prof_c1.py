"""The C1 desk trace (2000 steps) through rg_closed_loop_bisection (one k_loop_bisect launch) for
ncu; prints the rollouts x j* (cell-steps) of the trace."""
import sys
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop_bisection

out = run_closed_loop_bisection(rg.make_plant("surrogate-fc"), rg.ConstraintSet(-0.9, 0.9, anchor=0.0),
                                rg.DisturbanceModel.scaled(0.001, 3), rg.GovernorConfig(),
                                ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2))),
                                2000, 2024)
print("cell_steps", sum(r.diagnostics["sims_run"] for r, _ in out) * 256)
