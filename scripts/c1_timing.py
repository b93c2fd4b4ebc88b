"""C1 (BASELINE configs[0]): the nominal bisection governor's closed loop (desk profile,
2000 steps), ms per step on the device path, beside the reference on the host."""
import sys
import time
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop_bisection

plant = rg.make_plant("surrogate-fc")
box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
model = rg.DisturbanceModel.scaled(0.001, 3)
cfg = rg.GovernorConfig(j_star=256, n_kappa=8)
prof = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
run_closed_loop_bisection(plant, box, model, cfg, prof, 50, 2025)
t0 = time.perf_counter()
out = run_closed_loop_bisection(plant, box, model, cfg, prof, 2000, 2024)
print("device C1 (one kernel): %.4f ms/step" % ((time.perf_counter() - t0) / 2000 * 1e3))
run_closed_loop_bisection(plant, box, model, cfg, prof, 50, 2025, native=False)
t0 = time.perf_counter()
run_closed_loop_bisection(plant, box, model, cfg, prof, 2000, 2024, native=False)
print("device C1 (per-step bisection_rg): %.4f ms/step" % ((time.perf_counter() - t0) / 2000 * 1e3))
try:
    sys.path.insert(0, "oracle/_ref")
    import refgov  # noqa
    from refgov import harness as H
    print("reference importable")
except Exception as e:  # pragma: no cover
    print("reference not importable here:", e)
