"""Generate golden fixtures by running the REAL reference (`refgov`) in the build container.

Run (here only; /root/reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Every array is produced by the reference's own
public functions (numba kernels, glibc tanh, numpy tanh), never by this repo's
code.  The fixtures pin the CPU oracle (oracle/) and, on the GPU box, the CUDA
product.  Cases follow the reference's own tests: the bench snapshot
(harness.py:269-271), transient-binding trials (tests/test_acceptance.py:88-146),
overflow and out-of-bounds starts (kernels.py:52-53, 80-83), duplicate and
steady-state-pruned rows (governor.py:302-317), asymmetric and half-infinite
constraint sets (constraints.py:37-70), the bisection anchors
(tests/test_governor.py:217-297) and the desk-scale closed loops
(presets/desk-scale.json).
"""

from __future__ import annotations

import hashlib
import math
import sys
from pathlib import Path

import numpy as np

import refgov
from refgov import (
    ConstraintSet,
    DisturbanceModel,
    GovernorConfig,
    GovernorState,
    bisection_rg,
    derive_seed,
    load_config,
    robust_rg_parallel,
    robust_rg_sequential,
    run_closed_loop,
    sample_scenarios,
    update_setpoint,
)
from refgov import governor as G
from refgov import kernels as K
from refgov.constraints import tighten
from refgov.disturbance import _uniform_grid, counter_uniform, splitmix64

assert "/root/reference" in refgov.__file__, refgov.__file__

OUT = Path(__file__).resolve().parent / "golden.npz"
MASK = (1 << 64) - 1
rng = np.random.default_rng(20261018)
G_ = {}


def put(name, arr):
    G_[name] = np.asarray(arr)


def eq(v):
    return np.array([np.tanh(v), v, np.tanh(v) / 2.0])


plant = refgov.make_plant("surrogate-fc")
K.warmup()

# ---------------------------------------------------------------- RNG
put("sm_seed0", np.array([splitmix64((n * 0x9E3779B97F4A7C15) & MASK) for n in range(3)],
                         dtype=np.uint64))
zin = rng.integers(0, 2**63, size=64, dtype=np.int64).astype(np.uint64) * np.uint64(2) + \
    np.uint64(1)
put("sm_in", zin)
put("sm_out", np.array([splitmix64(int(z)) for z in zin], dtype=np.uint64))
coords = np.stack([
    rng.integers(0, 2**63, size=48, dtype=np.int64).astype(np.uint64) * np.uint64(2),
    rng.integers(0, 2**40, size=48, dtype=np.int64).astype(np.uint64),
    rng.integers(0, 4096, size=48, dtype=np.int64).astype(np.uint64),
    rng.integers(0, 3, size=48, dtype=np.int64).astype(np.uint64),
], axis=1)
put("cu_coords", coords)
put("cu_out", np.array([counter_uniform(*(int(c) for c in row)) for row in coords]))
labels = ["scenarios", "plant", "bench:serial:1000", "bench:multicore:1000", "ü-label"]
put("derive_labels", np.array(labels))
put("derive_out", np.array([derive_seed(2024, lb) for lb in labels] +
                           [derive_seed(2**64 - 1, "plant")], dtype=np.uint64))

ranges_asym = ((-0.003, 0.001), (0.0, 0.002), (-1e-4, 1e-4))
model_asym = DisturbanceModel(ranges=ranges_asym)
small = sample_scenarios(model_asym, 5, 9, seed=2**63 + 5)
put("scen_small", small.data)
put("scen_small_k0", _uniform_grid(2**64 - 3, 4, 6, 3, k0=1_000_000))
big = sample_scenarios(DisturbanceModel.scaled(0.001, 3), 1000, 257, seed=7)
put("scen_big_sha", np.frombuffer(hashlib.sha256(big.data.tobytes()).digest(), np.uint8))
put("scen_big_rows", big.data[[0, 1, 511, 999]])
# derive_seed(...) + t overflows 2**64 in run_closed_loop (harness.py:197)
wrap_seed = derive_seed(2024, "scenarios")
s_wrap = sample_scenarios(DisturbanceModel.scaled(0.001, 3), 3, 5, seed=(MASK - 1) + 5)
put("scen_wrap", s_wrap.data)

# ---------------------------------------------------------------- fills
box = ConstraintSet(-0.9, 0.9, anchor=0.0)
fill_cases = []


def add_fill(name, x0, v_prev, r, m_grid, n_sim, j_star, eps, ranges, seed, cset=box,
             prefix=False):
    model = DisturbanceModel(ranges=ranges)
    scen = sample_scenarios(model, n_sim, j_star + 1, seed=seed)
    grid = G.grid_kappas(m_grid)
    x0 = np.asarray(x0, dtype=np.float64)
    v_rows = np.array([update_setpoint(v_prev, r, float(k)) for k in grid])
    tight = tighten(cset, eps)
    ss = np.array([tight.contains(plant.steady_state_output(v)) for v in v_rows])
    # raw cell matrix for every row (no ss/dedup), straight from the numba kernel
    S = np.zeros((m_grid, n_sim), dtype=np.uint8)
    steps = np.zeros((m_grid, n_sim), dtype=np.int32)
    K.run_cells(plant, x0, v_rows, np.arange(m_grid), scen.data, j_star, cset.lower,
                cset.upper, S, steps, mode="serial")
    stats = {}
    P = G.fill_feasibility("serial", plant, x0, v_prev, r, grid, scen, cset, eps, j_star,
                           stats=stats)
    res = robust_rg_parallel(plant, x0, GovernorState(v_prev), r, cset, scen,
                             GovernorConfig(j_star=j_star, epsilon=eps, m_grid=m_grid,
                                            n_sim=n_sim, prefix_mode=prefix))
    pre = f"fill_{len(fill_cases)}_"
    fill_cases.append(name)
    put(pre + "x0", x0)
    put(pre + "scalars", np.array([v_prev, r, eps, cset.lower, cset.upper, cset.anchor,
                                   float(j_star), float(m_grid), float(n_sim),
                                   float(prefix)]))
    put(pre + "ranges", np.array(ranges, dtype=np.float64))
    put(pre + "seed", np.array([seed], dtype=np.uint64))
    put(pre + "S_all", S)
    put(pre + "steps_all", steps)
    put(pre + "ss_ok", ss)
    put(pre + "P", P)
    put(pre + "stats", np.array([stats["sims_run"], stats["early_terms"], stats["overflows"],
                                 stats["ss_pruned_rows"], stats["dedup_rows"]]))
    put(pre + "result", np.array([res.kappa_opt, res.v_applied, float(res.feasible)]))


sc = ((-0.001, 0.001),) * 3
add_fill("bench_snapshot", np.zeros(3), 0.0, 0.5, 32, 64, 256, 0.05, sc, 7)
for trial in range(10):
    v_prev = float(rng.uniform(-1.0, 1.0))
    r = float(rng.uniform(-2.5, 2.5))
    x0 = eq(v_prev) + rng.uniform(-0.05, 0.05, size=3)
    add_fill(f"transient_{trial}", x0, v_prev, r, 32, 48, 256, 0.05,
             ((-0.02, 0.02),) * 3, 9000 + trial)
add_fill("from_rest_r2.5", np.zeros(3), 0.0, 2.5, 32, 16, 256, 0.05, sc, 11)
add_fill("overflow", np.zeros(3), 0.0, 0.5, 8, 32, 16, 0.05, ((-2e6, 2e6),) * 3, 3)
add_fill("out_of_bounds_start", np.array([2.0, 0.0, 0.0]), 0.5, 0.6, 8, 8, 32, 0.05, sc, 4)
add_fill("edge_j1_m2_n1", np.zeros(3), 0.1, 0.2, 2, 1, 1, 0.05, sc, 5)
add_fill("duplicate_rows", eq(0.3), 0.3, 0.3, 16, 24, 64, 0.05, sc, 6)
add_fill("asymmetric_anchor", np.array([0.2, 0.1, 0.05]), 0.1, 1.7, 24, 32, 128, 0.1,
         ((-0.01, 0.005),) * 3, 8, cset=ConstraintSet(-0.5, 0.9, anchor=0.2))
add_fill("half_infinite", np.zeros(3), 0.0, 2.0, 16, 16, 128, 0.05, sc, 12,
         cset=ConstraintSet(-math.inf, 0.9, anchor=0.0))
add_fill("prefix_mode", np.zeros(3), 0.0, 2.5, 16, 16, 64, 0.05, ((-0.01, 0.01),) * 3, 3,
         prefix=True)
add_fill("paper_horizon", eq(-0.2) + 0.01, -0.2, 1.3, 32, 8, 1024, 0.05,
         ((-0.005, 0.005),) * 3, 77)
put("fill_names", np.array(fill_cases))

# ---------------------------------------------------------------- bisection
bis_cases = []


def add_bisect(name, x0, v_prev, r, n_sim, j_star, eps, ranges, seed, n_kappa=8, cset=box):
    model = DisturbanceModel(ranges=ranges)
    scen = sample_scenarios(model, n_sim, j_star + 1, seed=seed)
    x0 = np.asarray(x0, dtype=np.float64)
    tight = tighten(cset, eps)
    cfg = GovernorConfig(j_star=j_star, epsilon=eps, n_kappa=n_kappa, n_sim=n_sim)
    res = robust_rg_sequential(plant, x0, GovernorState(v_prev), r, cset, scen, cfg)
    per = np.array([G._bisect_kappa(plant, x0, v_prev, r, cset, eps, j_star, n_kappa,
                                    scen.data[k], tight) for k in range(n_sim)],
                   dtype=np.float64)
    # the per-scenario bisection path, replayed with the reference's own pieces
    paths = np.full((n_sim, n_kappa + 1, 2), np.nan)
    for k in range(n_sim):
        def feas(kappa):
            v = update_setpoint(v_prev, r, kappa)
            if not tight.contains(plant.steady_state_output(v)):
                return False
            st, _ = K.rollout_cell(plant, x0, v, scen.data[k], j_star, cset.lower,
                                   cset.upper)
            return st == K.CELL_OK
        ok = feas(1.0)
        paths[k, 0] = (1.0, ok)
        if not ok:
            lo, hi = 0.0, 1.0
            for it in range(n_kappa):
                kap = 0.5 * (lo + hi)
                ok = feas(kap)
                paths[k, it + 1] = (kap, ok)
                if ok:
                    lo = kap
                else:
                    hi = kap
    pre = f"bis_{len(bis_cases)}_"
    bis_cases.append(name)
    put(pre + "x0", x0)
    put(pre + "scalars", np.array([v_prev, r, eps, cset.lower, cset.upper, cset.anchor,
                                   float(j_star), float(n_kappa), float(n_sim)]))
    put(pre + "ranges", np.array(ranges, dtype=np.float64))
    put(pre + "seed", np.array([seed], dtype=np.uint64))
    put(pre + "result", np.array([res.kappa_opt, res.v_applied, float(res.feasible),
                                  res.diagnostics["sims_run"],
                                  res.diagnostics["early_terms"]]))
    put(pre + "per", per)
    put(pre + "paths", paths)


add_bisect("from_rest_r2.5", np.zeros(3), 0.0, 2.5, 8, 256, 0.05, sc, 1)
add_bisect("bench_r0.5", np.zeros(3), 0.0, 0.5, 16, 256, 0.05, sc, 2)
for trial in range(6):
    v_prev = float(rng.uniform(-1.0, 1.0))
    r = float(rng.uniform(-2.5, 2.5))
    x0 = eq(v_prev) + rng.uniform(-0.05, 0.05, size=3)
    add_bisect(f"transient_{trial}", x0, v_prev, r, 24, 256, 0.05, ((-0.02, 0.02),) * 3,
               4000 + trial)
add_bisect("nothing_feasible", np.array([2.0, 0.0, 0.0]), 0.5, 0.6, 4, 32, 0.05, sc, 3)
add_bisect("deep_nkappa", eq(0.4), 0.4, -2.2, 8, 128, 0.05, ((-0.01, 0.01),) * 3, 5,
           n_kappa=20)
put("bis_names", np.array(bis_cases))

# nominal bisection anchor quoted in SURVEY.md §8(c)
nb = bisection_rg(plant, np.zeros(3), GovernorState(0.0), 2.5, box, GovernorConfig())
put("nominal_anchor", np.array([nb.kappa_opt, nb.v_applied, float(nb.feasible),
                                nb.diagnostics["sims_run"], nb.diagnostics["early_terms"]]))

# ---------------------------------------------------------------- linear plant
# kernels.py:90-118 (_cell_lin) behind the same governors; shapes from the
# reference's oracle suite (oracle.py:201-232: n in 1..3, stable A, |dc gain| >= 0.2)
from refgov import LinearOraclePlant, linear_maximal_kappa
lin_cases = []


def add_linear(name, A, B, C, D, x0, v_prev, r, m_grid, n_sim, j_star, eps, mag, seed, cset):
    lp = LinearOraclePlant(A, B, C, D)
    n = lp.state_dim
    model = DisturbanceModel.scaled(mag, n)
    scen = sample_scenarios(model, n_sim, j_star + 1, seed=seed)
    x0 = np.asarray(x0, dtype=np.float64)
    grid = G.grid_kappas(m_grid)
    v_rows = np.array([update_setpoint(v_prev, r, float(k)) for k in grid])
    S = np.zeros((m_grid, n_sim), dtype=np.uint8)
    steps = np.zeros((m_grid, n_sim), dtype=np.int32)
    K.run_cells(lp, x0, v_rows, np.arange(m_grid), scen.data, j_star, cset.lower, cset.upper,
                S, steps, mode="serial")
    stats = {}
    P = G.fill_feasibility("serial", lp, x0, v_prev, r, grid, scen, cset, eps, j_star,
                           stats=stats)
    cfg = GovernorConfig(j_star=j_star, epsilon=eps, m_grid=m_grid, n_sim=n_sim)
    par = robust_rg_parallel(lp, x0, GovernorState(v_prev), r, cset, scen, cfg)
    seq = robust_rg_sequential(lp, x0, GovernorState(v_prev), r, cset, scen, cfg)
    nom = bisection_rg(lp, x0, GovernorState(v_prev), r, cset, cfg)
    pre = f"lin_{len(lin_cases)}_"
    lin_cases.append(name)
    put(pre + "A", lp.A)
    put(pre + "BCD", np.concatenate([lp.B, lp.C, [lp.D, lp.dc_gain]]))
    put(pre + "x0", x0)
    put(pre + "scalars", np.array([v_prev, r, eps, cset.lower, cset.upper, cset.anchor,
                                   float(j_star), float(m_grid), float(n_sim), mag]))
    put(pre + "seed", np.array([seed], dtype=np.uint64))
    put(pre + "S_all", S)
    put(pre + "steps_all", steps)
    put(pre + "P", P)
    put(pre + "stats", np.array([stats["sims_run"], stats["early_terms"], stats["overflows"],
                                 stats["ss_pruned_rows"], stats["dedup_rows"]]))
    put(pre + "results", np.array([
        par.kappa_opt, par.v_applied, float(par.feasible),
        seq.kappa_opt, seq.v_applied, float(seq.feasible), seq.diagnostics["sims_run"],
        seq.diagnostics["early_terms"],
        nom.kappa_opt, nom.v_applied, float(nom.feasible), nom.diagnostics["sims_run"],
        nom.diagnostics["early_terms"]]))


lbox = ConstraintSet(-0.9, 0.9)
# the reference's own known answer: kappa* = 0.81 (tests/test_oracle.py:27-34)
add_linear("scalar_kappa081", [[0.5]], [0.5], [1.0], 0.0, [0.0], 0.0, 1.0, 32, 8, 256, 0.1,
           1e-4, 1, lbox)
add_linear("two_state", [[0.85, 0.1], [0.0, 0.7]], [0.0, 0.3], [1.0, 0.0], 0.0, [0.0, 0.0],
           0.1, 1.0, 16, 24, 64, 0.1, 0.005, 4, lbox)
lrng = np.random.default_rng(424242)
for trial in range(6):
    while True:
        n = int(lrng.integers(1, 4))
        A = lrng.uniform(-1.0, 1.0, size=(n, n))
        rho = float(np.max(np.abs(np.linalg.eigvals(A))))
        if rho > 1e-12:
            A *= lrng.uniform(0.3, 0.95) / rho
        B = lrng.uniform(-1.0, 1.0, size=n)
        C = lrng.uniform(-1.0, 1.0, size=n)
        if abs(LinearOraclePlant(A, B, C).dc_gain) >= 0.2:
            break
    add_linear(f"random_{trial}_n{n}", A, B, C, float(lrng.uniform(-0.2, 0.2)),
               lrng.uniform(-0.3, 0.3, size=n), float(lrng.uniform(-0.5, 0.5)),
               float(lrng.uniform(-3, 3)), 32, 32, 128, 0.1, 0.01, 100 + trial,
               ConstraintSet(-1.0, 1.0))
add_linear("overflow_big_dist", [[0.9, 0.0, 0.0], [0.1, 0.5, 0.0], [0.0, 0.2, 0.3]],
           [1.0, 0.0, 0.0], [0.0, 0.0, 1.0], 0.0, [0.0, 0.0, 0.0], 0.0, 0.5, 8, 16, 16, 0.1,
           2e6, 9, ConstraintSet(-np.inf, 0.9))
put("lin_names", np.array(lin_cases))
put("lin_kappa_star_081", np.array([linear_maximal_kappa([[0.5]], [0.5], [1.0], np.zeros(1),
                                                          0.0, 1.0, lbox, 0.1, 256)]))

# ---------------------------------------------------------------- closed loops
setup = load_config({})
tight = tighten(setup.cset, setup.epsilon)
prof = setup.profile.schedule(setup.steps)
put("desk_profile", prof)

# C1: nominal bisection_rg substituted at harness.py:200 (the reference has no driver)
x = np.zeros(3)
state = GovernorState(0.0)
plant_seed = derive_seed(setup.seed, "plant")
lo_ = np.array([a for a, _ in setup.model.ranges])
span_ = np.array([b - a for a, b in setup.model.ranges])
d_true = lo_ + span_ * _uniform_grid(plant_seed, 1, setup.steps, 3)[0]
c1 = []
for t in range(setup.steps):
    res = bisection_rg(setup.plant, x, state, float(prof[t]), setup.cset, setup.governor)
    c1.append((res.kappa_opt, res.v_applied, float(res.feasible), float(x[0]),
               res.diagnostics["sims_run"], res.diagnostics["early_terms"]))
    x = setup.plant.step(x, res.v_applied) + d_true[t]
put("c1_trace", np.array(c1))

# reference closed loop with the grid governor, desk preset (n_sim=64, 2000 steps)
rec = run_closed_loop(setup.plant, setup.cset, setup.model, setup.governor, setup.profile,
                      setup.steps, setup.seed)
assert not rec.aborted
put("desk_grid_trace", np.array([[row[2], row[3], row[4], float(row[5])]
                                 for row in rec.rows]))
# truncated C3: n_sim = 1000 scenarios, first 40 steps of the desk trace (multicore)
setup3 = load_config({"governor": {"n_sim": 1000, "backend": "multicore"}})
rec3 = run_closed_loop(setup3.plant, setup3.cset, setup3.model, setup3.governor,
                       setup3.profile, 40, setup3.seed)
put("c3_trace40", np.array([[row[2], row[3], row[4], float(row[5])] for row in rec3.rows]))

# ---------------------------------------------------------------- tanh
xs = np.concatenate([
    rng.uniform(-3, 3, 4000), rng.uniform(-25, 25, 2000), rng.uniform(-1e-3, 1e-3, 500),
    np.ldexp(rng.uniform(0.5, 1, 200), rng.integers(-60, -20, 200)),
    np.array([0.0, -0.0, 1.0, -1.0, 22.0, -22.0, 21.999999999999996, 0.34657359027997264,
              0.5198603854199589, 19.0, 0.25, -0.25, 1e-300, 5e-324, np.inf, -np.inf]),
])
put("tanh_x", xs)
put("tanh_libm", np.array([math.tanh(float(v)) for v in xs]))
put("tanh_numpy", np.tanh(xs))
put("expm1_host", np.array([math.expm1(float(v)) for v in xs[:2000]]))

np.savez_compressed(OUT, **G_)
print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(G_)} arrays)", file=sys.stderr)
