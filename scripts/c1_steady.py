"""C1 loop variants: steady state (every step the kappa = 1 probe alone) and the desk trace, per
closed-loop step, with the passes per step inferred from cells and gating."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop_bisection

plant = rg.make_plant("surrogate-fc")
box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
model = rg.DisturbanceModel.scaled(0.001, 3)
cfg = rg.GovernorConfig(j_star=256, n_kappa=8)
for name, prof in (("steady r=0.4", [0.4] * 2000),
                   ("desk", ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2))))):
    run_closed_loop_bisection(plant, box, model, cfg, prof, 100, 5)
    t0 = time.perf_counter()
    out = run_closed_loop_bisection(plant, box, model, cfg, prof, 2000, 2024)
    dt = (time.perf_counter() - t0) / 2000 * 1e6
    dev = np.array([r.diagnostics["kernel_us"] for r, _ in out])
    cells = np.array([r.diagnostics["sims_run"] for r, _ in out])
    print(f"{name}: {dt:.1f} us per step (device {dev.mean():.1f}); cells per step {cells.mean():.2f}; "
          f"steps with 1 cell: {np.mean(dev[cells == 1]) if (cells == 1).any() else float('nan'):.1f} us",
          flush=True)
