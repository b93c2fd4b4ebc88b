"""Where a C3 closed-loop step's host time goes: cProfile of run_closed_loop over 600 steps
at 10k scenarios (after 100 warm-up steps), top entries by own time and cumulative."""
import cProfile
import pstats
import sys
import time
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop

plant = rg.make_plant("surrogate-fc")
box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
model = rg.DisturbanceModel.scaled(0.001, 3)
cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=10_000)
prof = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
run_closed_loop(plant, box, model, cfg, prof, 100, 2025)
t0 = time.perf_counter()
run_closed_loop(plant, box, model, cfg, prof, 600, 2024)
print("plain: %.4f ms/step" % ((time.perf_counter() - t0) / 600 * 1e3))
pr = cProfile.Profile()
pr.enable()
run_closed_loop(plant, box, model, cfg, prof, 600, 2024)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(25)
