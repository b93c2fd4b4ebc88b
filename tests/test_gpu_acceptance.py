"""The reference's release-gate criteria and governor properties, on the device path.

Each test restates one of the reference's own acceptance criteria
(`pkg/tests/test_acceptance.py`) or governor property tests
(`pkg/tests/test_governor.py`) with the CUDA backend in place of the
serial/multicore fills, so the guarantees the reference ships are checked on
the drop-in.  Where the reference compares two CPU backends, the device is
compared with the C oracle (oracle/, test infrastructure only) bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2510_08288_b200 as rg
from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop

pytestmark = pytest.mark.gpu

PLANT = rg.make_plant("surrogate-fc")
BOX = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
ORIGIN = np.zeros(3)
DESK_PROFILE = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))


def _equilibrium(v: float) -> np.ndarray:
    return np.array([np.tanh(v), v, np.tanh(v) / 2.0])


# ----------------------------------------------------------------- acceptance criteria

def test_criterion_3_device_determinism(orc):
    """test_acceptance.py:88-112: every backend's P is bit-identical to serial.

    Here: the device fill equals the oracle's serial fill, call after call, for
    host-staged and device-generated copies of the same scenarios.
    """
    rng = np.random.default_rng(31)
    model = rg.DisturbanceModel.scaled(0.001, 3)
    grid = rg.grid_kappas(32)
    tlo, thi = orc.tighten(-0.9, 0.9, 0.0, 0.05)
    for trial in range(20):
        v_prev = float(rng.uniform(-1.0, 1.0))
        r = float(rng.uniform(-2.5, 2.5))
        x0 = _equilibrium(v_prev) + rng.uniform(-0.05, 0.05, size=3)
        gen = rg.sample_scenarios(model, 256, 257, seed=9000 + trial, device=0)
        host = rg.ScenarioSet(gen.data.copy())
        ref, _, _, _ = orc.fill_feasibility(0.01, x0, v_prev, r, grid, host.data, -0.9, 0.9,
                                            tlo, thi, 256)
        for scen in (host, gen, host):
            P = rg.fill_feasibility("cuda", PLANT, x0, v_prev, r, grid, scen, BOX, 0.05, 256)
            assert np.array_equal(P, ref), trial
            assert rg.extract_kappa_opt(P) == orc.extract_kappa_opt(ref)


def test_criterion_4_robustness_monotonicity(orc):
    """test_acceptance.py:115-146: kappa never grows as nested scenario sets grow."""
    rng = np.random.default_rng(44)
    model = rg.DisturbanceModel.scaled(0.02, 3)
    tlo, thi = orc.tighten(-0.9, 0.9, 0.0, 0.05)
    dropped = 0
    for trial in range(20):
        v_prev = float(rng.uniform(-0.5, 0.5))
        r = float(rng.uniform(-2.0, 2.0))
        x0 = _equilibrium(v_prev)
        big = rg.sample_scenarios(model, 256, 257, seed=5000 + trial)
        kappas = []
        for n in (16, 64, 256):
            scen = rg.sample_scenarios(model, n, 257, seed=5000 + trial)
            assert np.array_equal(scen.data, big.data[:n])
            cfg = rg.GovernorConfig(j_star=256, n_sim=n, m_grid=32)
            res = rg.robust_rg_parallel(PLANT, x0, rg.GovernorState(v_prev), r, BOX, scen, cfg)
            k, v, feas, _, _, _ = orc.grid_step(0.01, x0, v_prev, r, 32, scen.data, -0.9, 0.9,
                                                tlo, thi, 256)
            assert (res.kappa_opt, res.v_applied, res.feasible) == (k, v, feas)
            kappas.append(res.kappa_opt if res.feasible else -1.0)
        assert kappas[0] >= kappas[1] >= kappas[2], (trial, kappas)
        dropped += kappas[0] > kappas[2]
    assert dropped >= 1   # the property is exercised, not passed by ties


def test_criterion_5_closed_loop_enforcement():
    """test_acceptance.py:149-169: desk-scale loop, 10 seeds x 2000 steps.

    Without the governor the true plant leaves the output band on every seed;
    with the device governor it never does.
    """
    cfg = rg.GovernorConfig()   # desk-scale governor: j*=256, M=32, n_sim=64
    model = rg.DisturbanceModel.scaled(0.001, 3)
    off_viol, on_viol = [], []
    for seed in range(3001, 3011):
        off = run_closed_loop(PLANT, BOX, model, cfg, DESK_PROFILE, 2000, seed,
                              governor_on=False)
        on = run_closed_loop(PLANT, BOX, model, cfg, DESK_PROFILE, 2000, seed)
        assert not on.aborted and len(on.rows) == 2000
        off_viol.append(off.violations(BOX))
        on_viol.append(on.violations(BOX))
    assert all(v >= 1 for v in off_viol), off_viol
    assert all(v == 0 for v in on_viol), on_viol


def test_criterion_6_zero_scenario_collapse():
    """test_acceptance.py:172-211: one zero scenario = the disturbance-free grid search.

    The plain search runs straight off the host plant methods (numpy tanh), as
    in the reference test.
    """
    rng = np.random.default_rng(66)
    j_star = 64
    grid = rg.grid_kappas(32)
    tight = rg.tighten(BOX, 0.05)
    cfg = rg.GovernorConfig(j_star=j_star, n_sim=1, m_grid=32)

    def plain_grid_kappa(x0, v_prev, r):
        best = None
        for kappa in grid:
            v = rg.update_setpoint(v_prev, r, float(kappa))
            if not tight.contains(PLANT.steady_state_output(v)):
                continue
            x = x0.copy()
            feasible = BOX.contains(PLANT.output(x, v))
            for _ in range(j_star):
                if not feasible:
                    break
                x = PLANT.step(x, v)
                feasible = BOX.contains(PLANT.output(x, v))
            if feasible:
                best = float(kappa)
        return best

    for _ in range(25):
        v_prev = float(rng.uniform(-1.0, 1.0))
        r = float(rng.uniform(-2.5, 2.5))
        x0 = _equilibrium(v_prev) + rng.uniform(-0.1, 0.1, size=3)
        res = rg.robust_rg_parallel(PLANT, x0, rg.GovernorState(v_prev), r, BOX,
                                    rg.zero_scenarios(3, j_star + 1), cfg)
        robust = res.kappa_opt if res.feasible else None
        assert robust == plain_grid_kappa(x0, v_prev, r), (v_prev, r)


# ----------------------------------------------------------------- governor properties

def test_bisection_short_circuits_on_feasible_full_step():
    """test_governor.py:217-223: kappa = 1 feasible -> one rollout."""
    res = rg.bisection_rg(PLANT, ORIGIN, rg.GovernorState(0.0), 0.3, BOX,
                          rg.GovernorConfig(j_star=64, n_sim=1))
    assert (res.kappa_opt, res.v_applied, res.feasible) == (1.0, 0.3, True)
    assert res.diagnostics["sims_run"] == 1


def test_bisection_holds_when_nothing_feasible():
    """test_governor.py:239-246: y outside the band at step 0 -> hold."""
    state = rg.GovernorState(0.5)
    res = rg.bisection_rg(PLANT, np.array([2.0, 0.0, 0.0]), state, 0.6, BOX,
                          rg.GovernorConfig(j_star=32, n_sim=1))
    assert (res.kappa_opt, res.v_applied, res.feasible) == (0.0, 0.5, False)


def test_sequential_takes_worst_scenario():
    """test_governor.py:259-271: Alg. 2 = min over one-scenario searches."""
    scen = rg.sample_scenarios(rg.DisturbanceModel.scaled(0.02, 3), 8, 65, seed=6)
    res = rg.robust_rg_sequential(PLANT, ORIGIN, rg.GovernorState(0.0), 2.5, BOX, scen,
                                  rg.GovernorConfig(j_star=64, n_sim=8))
    per = [rg.robust_rg_sequential(PLANT, ORIGIN, rg.GovernorState(0.0), 2.5, BOX,
                                   rg.ScenarioSet(scen.data[k:k + 1]),
                                   rg.GovernorConfig(j_star=64, n_sim=1)).kappa_opt
           for k in range(8)]
    assert res.kappa_opt == min(per)
    joint = rg.robust_rg_joint(PLANT, ORIGIN, rg.GovernorState(0.0), 2.5, BOX, scen,
                               rg.GovernorConfig(j_star=64, n_sim=8))
    assert joint.kappa_opt == res.kappa_opt


def test_parallel_kappa_is_on_grid_and_below_bisection():
    """test_governor.py:289-297, plus the measured anchors of SURVEY.md §8(c)."""
    rp = rg.robust_rg_parallel(PLANT, ORIGIN, rg.GovernorState(0.0), 2.5, BOX,
                               rg.zero_scenarios(3, 257),
                               rg.GovernorConfig(j_star=256, n_sim=1, m_grid=32))
    rb = rg.bisection_rg(PLANT, ORIGIN, rg.GovernorState(0.0), 2.5, BOX,
                         rg.GovernorConfig(j_star=256, n_sim=1))
    assert rp.kappa_opt in rg.grid_kappas(32)
    assert rp.kappa_opt <= rb.kappa_opt + 1.0 / 31.0
    assert rp.kappa_opt == 15 / 31 and rp.v_applied == 1.2096774193548387
    assert rb.kappa_opt == 0.5078125


def test_parallel_infeasible_hold_keeps_setpoint():
    """test_governor.py:300-308."""
    state = rg.GovernorState(0.7)
    res = rg.robust_rg_parallel(PLANT, np.array([2.0, 0.0, 0.0]), state, 1.0, BOX,
                                rg.zero_scenarios(3, 33),
                                rg.GovernorConfig(j_star=32, n_sim=1, m_grid=8,
                                                  infeasible_policy="hold"))
    assert (res.kappa_opt, res.v_applied, res.feasible) == (0.0, 0.7, False)
    assert state.v_prev == 0.7


def test_parallel_prefix_mode_is_never_less_conservative():
    """test_governor.py:320-326."""
    scen = rg.sample_scenarios(rg.DisturbanceModel.scaled(0.01, 3), 16, 65, seed=3)
    r0 = rg.robust_rg_parallel(PLANT, ORIGIN, rg.GovernorState(0.0), 2.5, BOX, scen,
                               rg.GovernorConfig(j_star=64, n_sim=16, m_grid=16))
    r1 = rg.robust_rg_parallel(PLANT, ORIGIN, rg.GovernorState(0.0), 2.5, BOX, scen,
                               rg.GovernorConfig(j_star=64, n_sim=16, m_grid=16,
                                                 prefix_mode=True))
    assert r1.kappa_opt <= r0.kappa_opt


def test_parallel_nested_scenarios_shrink_kappa():
    """test_governor.py:329-339."""
    big = rg.sample_scenarios(rg.DisturbanceModel.scaled(0.05, 3), 64, 65, seed=17)
    kappas = [rg.robust_rg_parallel(PLANT, ORIGIN, rg.GovernorState(0.0), 2.5, BOX,
                                    big.prefix(n),
                                    rg.GovernorConfig(j_star=64, n_sim=n, m_grid=32)).kappa_opt
              for n in (4, 16, 64)]
    assert kappas[0] >= kappas[1] >= kappas[2]
