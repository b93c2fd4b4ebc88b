"""The native closed loop (rg_closed_loop: grid step, kappa, v_t and the true plant with
the library's numpy-tanh, per step in C) against the per-step Python loop
(run_closed_loop(native=False)), which is pinned to the reference's golden traces: equal
rows, diagnostics, abort reasons and errors."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2510_08288_b200 as rg
from paper_2510_08288_b200.errors import InfeasibleError
from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop

pytestmark = pytest.mark.gpu

PLANT = rg.make_plant("surrogate-fc")
BOX = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
DESK = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))


def _same(a, b):
    assert a.rows == b.rows  # (t, r, v, y, kappa, feasible, wall_us): wall_us differs
    assert a.diag_rows == b.diag_rows
    assert (a.aborted, a.abort_reason) == (b.aborted, b.abort_reason)


def _strip_wall(rec):
    rec.rows = [r[:6] for r in rec.rows]
    rec.diag_rows = [",".join(d.split(",")[:6]) for d in rec.diag_rows]
    return rec


@pytest.mark.parametrize("n_sim,steps,seed", [(1000, 700, 2024), (10_000, 450, 77),
                                              (300, 1200, 5)])
def test_native_loop_equals_python_loop(n_sim, steps, seed):
    model = rg.DisturbanceModel.scaled(0.001, 3)
    cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=n_sim)
    prof = DESK if steps < 1000 else ReferenceProfile(((0, 0.4), (300, 2.5), (700, -2.5),
                                                       (1000, 0.2)))
    nat = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, prof, steps, seed))
    py = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, prof, steps, seed, native=False))
    _same(nat, py)
    assert not nat.aborted and len(nat.rows) == steps


def test_native_loop_transients_prefix_mode_and_start_state():
    """Larger disturbances, prefix extraction, j* = 64, and a start outside the output
    bounds with v0 != 0: the first steps have no feasible row and hold the setpoint."""
    model = rg.DisturbanceModel.scaled(0.02, 3)
    cfg = rg.GovernorConfig(j_star=64, m_grid=16, n_sim=2000, prefix_mode=True)
    prof = np.concatenate([np.full(60, 2.0), np.full(60, -2.4), np.full(80, 0.7)])
    x0 = np.array([0.95, -0.5, 0.1])
    nat = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, prof, 200, 31, x0=x0, v0=-0.5))
    py = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, prof, 200, 31, x0=x0, v0=-0.5,
                                     native=False))
    _same(nat, py)
    assert not nat.rows[0][5] and any(r[5] for r in nat.rows)  # held, then feasible


def test_native_loop_aborts_like_the_python_loop():
    model = rg.DisturbanceModel.scaled(0.02, 3)
    cfg = rg.GovernorConfig(j_star=32, m_grid=8, n_sim=64)
    # the plant's integration overflow at step 0 (|x1| beyond 1e6 after the RK4 step)
    x0 = np.array([1.5e6, 0.0, 0.0])
    a = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, [0.4] * 5, 5, 3, x0=x0))
    b = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, [0.4] * 5, 5, 3, x0=x0,
                                    native=False))
    _same(a, b)
    assert a.aborted and "integration overflow in state 0" in a.abort_reason
    # the state leaving the box after the disturbance: x2 at the edge, held setpoint 1e6
    x0 = np.array([0.0, 1e6 - 1e-4, 0.0])
    a = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, [1e6] * 20, 20, 4, x0=x0, v0=1e6))
    b = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, [1e6] * 20, 20, 4, x0=x0, v0=1e6,
                                    native=False))
    _same(a, b)
    assert a.aborted and "left the operating box" in a.abort_reason


def test_native_loop_infeasible_error_policy():
    model = rg.DisturbanceModel.scaled(0.001, 3)
    cfg = rg.GovernorConfig(j_star=32, m_grid=8, n_sim=64, infeasible_policy="error")
    x0 = np.array([0.95, 0.0, 0.0])  # out of the output bounds: nothing is feasible
    with pytest.raises(InfeasibleError):
        run_closed_loop(PLANT, BOX, model, cfg, [0.4] * 3, 3, 1, x0=x0)
    with pytest.raises(InfeasibleError):
        run_closed_loop(PLANT, BOX, model, cfg, [0.4] * 3, 3, 1, x0=x0, native=False)


@pytest.mark.parametrize("case", ["desk_10k", "transient_prefix", "held_start", "small_grid"])
def test_device_loop_equals_per_step_loop(case):
    """rg_closed_loop runs the whole trace as one cooperative kernel (k_loop_ts: block 0
    extracts the row, steps the true plant with numpy's tanh on the device and plans the
    next rows between grid barriers); with "no_device_loop" it launches one grid step per
    closed-loop step from the host.  Same rows, diagnostics and aborts.  The desk case at 10k
    crosses the profile's jumps, where many rows are live and a step takes several passes of
    three units per block."""
    from paper_2510_08288_b200 import _capi

    ctx = _capi.context(0)
    x0, v0, prefix = None, 0.0, False
    if case == "desk_10k":
        model = rg.DisturbanceModel.scaled(0.001, 3)
        cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=10_000)
        prof = ReferenceProfile(((0, 0.4), (40, 2.5), (120, -2.5), (200, 0.2)))
        steps, seed = 260, 2024
    elif case == "transient_prefix":
        model = rg.DisturbanceModel.scaled(0.02, 3)
        cfg = rg.GovernorConfig(j_star=64, m_grid=16, n_sim=3000, prefix_mode=True)
        prof = np.concatenate([np.full(50, 2.0), np.full(50, -2.4), np.full(60, 0.7)])
        steps, seed = 160, 31
    elif case == "held_start":
        model = rg.DisturbanceModel.scaled(0.02, 3)
        cfg = rg.GovernorConfig(j_star=64, m_grid=64, n_sim=700)
        prof = np.concatenate([np.full(60, 2.0), np.full(60, -0.4)])
        steps, seed = 120, 5
        x0, v0 = np.array([0.95, -0.5, 0.1]), -0.5
    else:
        model = rg.DisturbanceModel.scaled(0.005, 3)
        cfg = rg.GovernorConfig(j_star=1, m_grid=2, n_sim=1)
        prof = np.concatenate([np.full(30, 1.5), np.full(30, -1.5)])
        steps, seed = 60, 9
    kw = {} if x0 is None else {"x0": x0, "v0": v0}
    dev = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, prof, steps, seed, **kw))
    assert ctx.get_option("last_loop_device") == 1
    ctx.set_option("no_device_loop", 1)
    try:
        host = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, prof, steps, seed, **kw))
        assert ctx.get_option("last_loop_device") == 0
    finally:
        ctx.set_option("no_device_loop", 0)
    _same(dev, host)
    assert len(dev.rows) == steps


def _c1_rows(rows):
    return [(r.kappa_opt, r.v_applied, r.feasible, y, r.diagnostics["sims_run"],
             r.diagnostics["early_terms"]) for r, y in rows]


@pytest.mark.parametrize("case", ["desk", "transient", "held_start", "deep"])
def test_device_bisection_loop_equals_per_step_loop(case):
    """C1's nominal bisection loop as one device kernel (rg_closed_loop_bisection: every
    candidate's rollout on the time-split passes of one block, the true plant with numpy's
    tanh on the device) against the per-step loop over bisection_rg: the same kappa, v_t,
    found, y_t, rollout and early counts every step."""
    from paper_2510_08288_b200.harness import run_closed_loop_bisection

    model = rg.DisturbanceModel.scaled(0.001, 3)
    x0, v0 = None, 0.0
    if case == "desk":
        cfg = rg.GovernorConfig()
        prof = ReferenceProfile(((0, 0.4), (40, 2.5), (140, -2.5), (240, 0.2)))
        steps, seed = 300, 2024
    elif case == "transient":
        model = rg.DisturbanceModel.scaled(0.02, 3)
        cfg = rg.GovernorConfig(j_star=64, n_kappa=5)
        prof = np.concatenate([np.full(40, 2.0), np.full(40, -2.4), np.full(40, 0.7)])
        steps, seed = 120, 31
    elif case == "held_start":
        cfg = rg.GovernorConfig(j_star=32, n_kappa=3)
        prof = np.concatenate([np.full(30, 2.0), np.full(30, -0.4)])
        steps, seed = 60, 5
        x0, v0 = np.array([0.95, -0.5, 0.1]), -0.5
    else:
        cfg = rg.GovernorConfig(j_star=1, n_kappa=20)
        prof = np.concatenate([np.full(20, 1.5), np.full(20, -1.5)])
        steps, seed = 40, 9
    kw = {} if x0 is None else {"x0": x0, "v0": v0}
    dev = run_closed_loop_bisection(PLANT, BOX, model, cfg, prof, steps, seed, **kw)
    host = run_closed_loop_bisection(PLANT, BOX, model, cfg, prof, steps, seed, native=False,
                                     **kw)
    assert _c1_rows(dev) == _c1_rows(host)
    assert len(dev) == steps


def test_device_bisection_loop_overflow_raises_like_the_plant():
    from paper_2510_08288_b200.errors import IntegrationOverflowError
    from paper_2510_08288_b200.harness import run_closed_loop_bisection

    cfg = rg.GovernorConfig(j_star=16, n_kappa=3)
    x0 = np.array([1.5e6, 0.0, 0.0])
    msgs = []
    for native in (None, False):
        with pytest.raises(IntegrationOverflowError) as e:
            run_closed_loop_bisection(PLANT, BOX, rg.DisturbanceModel.scaled(0.001, 3), cfg,
                                      [0.4] * 5, 5, 3, x0=x0, native=native)
        msgs.append((str(e.value), e.value.state_index))
    assert msgs[0] == msgs[1]


def test_large_scenario_sets_keep_the_per_step_loop():
    """Above one wave of the time-split form for a single row (ceil(n_sim / 32) > 3 x SMs)
    rg_closed_loop launches a grid step per closed-loop step (k_grid for the big steps) rather
    than many passes per step; the rows still equal the Python loop's."""
    from paper_2510_08288_b200 import _capi

    import torch

    ctx = _capi.context(0)
    n = 32 * 3 * torch.cuda.get_device_properties(0).multi_processor_count + 64
    cfg = rg.GovernorConfig(j_star=64, m_grid=16, n_sim=n)
    prof = np.concatenate([np.full(15, 0.4), np.full(15, 2.0)])
    model = rg.DisturbanceModel.scaled(0.001, 3)
    nat = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, prof, 30, 12))
    assert ctx.get_option("last_loop_device") == 0
    py = _strip_wall(run_closed_loop(PLANT, BOX, model, cfg, prof, 30, 12, native=False))
    _same(nat, py)
