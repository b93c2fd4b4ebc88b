"""A 200-step desk closed loop at 10k scenarios through rg_closed_loop (one k_loop_ts launch)
for ncu; prints the cell-steps of the trace (the sims_run x j* sum)."""
import sys
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=n)
rec = run_closed_loop(rg.make_plant("surrogate-fc"), rg.ConstraintSet(-0.9, 0.9, anchor=0.0),
                      rg.DisturbanceModel.scaled(0.001, 3), cfg,
                      ReferenceProfile(((0, 0.4), (400, 2.5))), 200, 2024)
print("cell_steps", sum(int(d.split(",")[4]) for d in rec.diag_rows) * 256)
