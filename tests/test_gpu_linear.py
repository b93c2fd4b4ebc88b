"""Linear plants on the device (kernels.py:90-118 behind the governors): bit-exact
against the reference's golden outputs, and the reference's closed-form
acceptance criteria 1 and 2 (tests/test_acceptance.py:45-85)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
from conftest import GOLDEN, lin_case

pytestmark = pytest.mark.gpu

with np.load(GOLDEN) as _z:
    N_LIN = len(_z["lin_names"])


def _plant(c):
    return rg.LinearOraclePlant(c["A"], c["B"], c["C"], c["D"])


@pytest.mark.parametrize("source", ["dense", "generated"])
@pytest.mark.parametrize("idx", range(N_LIN))
def test_linear_governors_match_reference(golden, idx, source):
    c = lin_case(golden, idx)
    plant = _plant(c)
    n = plant.state_dim
    cset = rg.ConstraintSet(c["lower"], c["upper"], c["anchor"])
    model = rg.DisturbanceModel.scaled(c["mag"], n)
    scen = rg.sample_scenarios(model, c["n_sim"], c["j_star"] + 1, c["seed"])
    if source == "dense":
        scen = rg.ScenarioSet(scen.data)
    stats = {}
    P = rg.fill_feasibility("cuda", plant, c["x0"], c["v_prev"], c["r"],
                            rg.grid_kappas(c["m_grid"]), scen, cset, c["eps"], c["j_star"],
                            stats=stats)
    assert np.array_equal(P, c["P"]), c["name"]
    assert [stats[k] for k in ("sims_run", "early_terms", "overflows", "ss_pruned_rows",
                               "dedup_rows")] == [int(v) for v in c["stats"]]
    cfg = rg.GovernorConfig(j_star=c["j_star"], epsilon=c["eps"], m_grid=c["m_grid"],
                            n_sim=c["n_sim"])
    par = rg.robust_rg_parallel(plant, c["x0"], rg.GovernorState(c["v_prev"]), c["r"], cset,
                                scen, cfg)
    seq = rg.robust_rg_sequential(plant, c["x0"], rg.GovernorState(c["v_prev"]), c["r"], cset,
                                  scen, cfg)
    nom = rg.bisection_rg(plant, c["x0"], rg.GovernorState(c["v_prev"]), c["r"], cset, cfg)
    got = [par.kappa_opt, par.v_applied, float(par.feasible),
           seq.kappa_opt, seq.v_applied, float(seq.feasible), seq.diagnostics["sims_run"],
           seq.diagnostics["early_terms"],
           nom.kappa_opt, nom.v_applied, float(nom.feasible), nom.diagnostics["sims_run"],
           nom.diagnostics["early_terms"]]
    assert got == [float(v) for v in c["results"]], c["name"]


def test_linear_cells_rng_path(golden, orc):
    c = lin_case(golden, 1)
    plant = _plant(c)
    n = plant.state_dim
    m = rg.DisturbanceModel.scaled(c["mag"], n)
    ctx = _capi.context(0)
    tight = rg.tighten(rg.ConstraintSet(c["lower"], c["upper"]), c["eps"])
    lin = _capi.make_linear(plant, tight.lower, tight.upper)
    prob = _capi.Problem(1.0, c["lower"], c["upper"], 0, 0, c["j_star"], 0)
    grid = rg.grid_kappas(c["m_grid"])
    v_rows = np.array([rg.update_setpoint(c["v_prev"], c["r"], float(k)) for k in grid])
    S = np.zeros((c["m_grid"], c["n_sim"]), np.uint8)
    steps = np.zeros_like(S, dtype=np.int32)
    ctx.fill_linear(lin, prob, c["x0"], v_rows, np.arange(c["m_grid"], dtype=np.int32), None,
                    c["n_sim"], _capi.make_scenarios(c["seed"], 0, c["n_sim"], m.lo, m.span), S,
                    steps)
    assert np.array_equal(S, c["S_all"]) and np.array_equal(steps, c["steps_all"])


def test_linear_bisection_known_answer():
    # reference tests/test_governor.py:226-236: kappa* = 0.81, bracket 2^-8
    plant = rg.LinearOraclePlant([[0.5]], [0.5], [1.0])
    cset = rg.ConstraintSet(-0.9, 0.9)
    cfg = rg.GovernorConfig(j_star=256, epsilon=0.1, n_kappa=8, n_sim=1)
    res = rg.bisection_rg(plant, np.zeros(1), rg.GovernorState(0.0), 1.0, cset, cfg)
    assert res.kappa_opt <= 0.81 + 1e-9 and 0.81 - res.kappa_opt <= 0.5**8 + 1e-9


def _random_case(rng, j_star, orc):
    while True:
        n = int(rng.integers(1, 4))
        A = rng.uniform(-1.0, 1.0, size=(n, n))
        rho = float(np.max(np.abs(np.linalg.eigvals(A))))
        if rho > 1e-12:
            A *= rng.uniform(0.3, 0.95) / rho
        B = rng.uniform(-1.0, 1.0, size=n)
        C = rng.uniform(-1.0, 1.0, size=n)
        plant = rg.LinearOraclePlant(A, B, C)
        if abs(plant.dc_gain) < 0.2:
            continue
        v_prev, r = float(rng.uniform(-0.5, 0.5)), float(rng.uniform(-3.0, 3.0))
        x0 = rng.uniform(-0.3, 0.3, size=n)
        tlo, thi = orc.tighten(-1.0, 1.0, 0.0, 0.1)
        if orc.linear_maximal_kappa(A, B, C, 0.0, x0, v_prev, v_prev, -1.0, 1.0, tlo, thi,
                                    j_star) is None:
            continue
        return plant, x0, v_prev, r, tlo, thi


def test_acceptance_criteria_1_and_2_on_device(orc):
    """Grid within one slot below the closed form; bisection inside (k* - 2^-8, k*]."""
    rng = np.random.default_rng(20260815)
    cset = rg.ConstraintSet(-1.0, 1.0)
    j_star = 128
    for _ in range(60):
        plant, x0, v_prev, r, tlo, thi = _random_case(rng, j_star, orc)
        k_star = orc.linear_maximal_kappa(plant.A, plant.B, plant.C, 0.0, x0, v_prev, r, -1.0,
                                          1.0, tlo, thi, j_star)
        cfg = rg.GovernorConfig(j_star=j_star, epsilon=0.1, m_grid=32, n_sim=1)
        zero = rg.zero_scenarios(plant.state_dim, j_star + 1)
        grid = rg.robust_rg_parallel(plant, x0, rg.GovernorState(v_prev), r, cset, zero, cfg)
        bis = rg.bisection_rg(plant, x0, rg.GovernorState(v_prev), r, cset, cfg)
        assert grid.feasible and bis.feasible
        assert grid.kappa_opt <= k_star + 1e-9 and k_star - grid.kappa_opt <= 1 / 31 + 1e-3
        assert bis.kappa_opt <= k_star + 1e-9 and k_star - bis.kappa_opt <= 0.5**8 + 1e-9
