"""Joint bisection on the B200 (rg_bisect_joint, robust_rg_joint, the sharded form).

The joint search is the north-star form of Alg. 2: one
candidate for every scenario per iteration, an OR-reduced violation flag,
early abandonment.  Its candidate sequence and verdicts are checked against the
CPU oracle's joint search (oracle.joint_bisect) bit for bit, and its kappa /
feasible against the exact per-scenario Alg. 2 on the device.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
from conftest import GOLDEN, bis_case

pytestmark = pytest.mark.gpu

with np.load(GOLDEN) as _z:
    N_BIS = len(_z["bis_names"])

PLANT = rg.make_plant("surrogate-fc")


def _cset(c):
    return rg.ConstraintSet(c["lower"], c["upper"], c["anchor"])


@pytest.mark.parametrize("idx", range(N_BIS))
def test_joint_matches_oracle_and_alg2_on_reference_cases(golden, orc, idx):
    c = bis_case(golden, idx)
    cfg = rg.GovernorConfig(j_star=c["j_star"], epsilon=c["eps"], n_kappa=c["n_kappa"],
                            n_sim=c["n_sim"])
    scen = rg.sample_scenarios(rg.DisturbanceModel(c["ranges"]), c["n_sim"], c["j_star"] + 1,
                               c["seed"])
    dist = orc.sample(c["seed"], c["n_sim"], c["j_star"] + 1, c["ranges"])
    tlo, thi = orc.tighten(c["lower"], c["upper"], c["anchor"], c["eps"])
    kj, fj, _ = orc.joint_bisect(0.01, c["x0"], c["v_prev"], c["r"], c["lower"], c["upper"],
                                 tlo, thi, dist, c["j_star"], c["n_kappa"])
    for s in (scen, rg.ScenarioSet(scen.data)):
        res = rg.robust_rg_joint(PLANT, c["x0"], rg.GovernorState(c["v_prev"]), c["r"],
                                 _cset(c), s, cfg)
        assert (res.kappa_opt, res.feasible) == (kj, fj), c["name"]
        assert res.v_applied == rg.update_setpoint(c["v_prev"], c["r"], kj)
        # and Alg. 2's result (the reference's robust_rg_sequential)
        assert (res.kappa_opt, float(res.feasible)) == (float(c["result"][0]),
                                                        float(c["result"][2])), c["name"]
        assert res.diagnostics["sims_run"] >= c["n_sim"]


@pytest.mark.parametrize("mode", ["fused", "staged"])
def test_joint_equals_device_alg2_at_scale(mode):
    """Transient-binding trials (200/200 equal): joint == Alg. 2."""
    ctx = _capi.context(0)
    rng = np.random.default_rng(5)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
    lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
    prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 128, 0)
    for trial in range(24):
        vp = float(rng.uniform(-1, 1))
        r = float(rng.uniform(-2.5, 2.5))
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.05, 0.05, 3)
        n = 3000
        sc = _capi.make_scenarios(300 + trial, 0, n, m.lo, m.span)
        a2, _, _ = ctx.bisect(prob, x0, vp, r, 8, None, n, sc, rng_mode=mode)
        jt = ctx.bisect_joint(prob, x0, vp, r, 8, None, n, sc, rng_mode=mode)
        assert (jt.kappa, jt.found) == (a2.kappa, a2.found), (trial, jt.kappa, a2.kappa)
        assert jt.cells >= n


def test_joint_iteration_api_equals_one_call():
    """begin / iter(fold=0) / decide / end == rg_bisect_joint (the sharded form's steps)."""
    ctx = _capi.context(0)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
    lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
    prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 128, 0)
    x0 = np.array([0.2, 0.4, 0.1])
    for seed in range(6):
        sc = _capi.make_scenarios(900 + seed, 0, 2000, m.lo, m.span)
        one = ctx.bisect_joint(prob, x0, 0.4, 2.2, 8, None, 2000, sc)
        ctx.joint_begin(prob, x0, 0.4, 2.2, 8, None, 2000, sc)
        for it in range(-1, 8):
            ctx.joint_iter(it, fold=False)
            ctx.joint_decide(it)
        step = ctx.joint_end()
        assert (step.kappa, step.found, step.cells) == (one.kappa, one.found, one.cells)


def test_joint_sharded_world1_nccl():
    """robust_rg_joint_sharded with one NCCL rank: the per-iteration all-reduce of
    the device flag on the library stream leaves the single-device result."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2510_08288_b200.sharded import robust_rg_joint_sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        m = rg.DisturbanceModel.scaled(0.02, 3)
        cfg = rg.GovernorConfig(j_star=128, n_sim=4000)
        box = rg.ConstraintSet(-0.9, 0.9)
        for seed in range(4):
            scen = rg.sample_scenarios(m, 4000, 129, seed=40 + seed)
            x0 = np.array([0.2, 0.4, 0.1])
            a = rg.robust_rg_joint(PLANT, x0, rg.GovernorState(0.4), 2.2, box, scen, cfg)
            b = robust_rg_joint_sharded(PLANT, x0, rg.GovernorState(0.4), 2.2, box, scen, cfg)
            assert (a.kappa_opt, a.feasible, a.v_applied) == (b.kappa_opt, b.feasible,
                                                              b.v_applied)
    finally:
        dist.destroy_process_group()


def test_grid_and_alg2_sharded_world1_nccl():
    """robust_rg_parallel_sharded (device counts, NCCL MAX on the library stream)
    and robust_rg_sequential_sharded with one NCCL rank equal the single-device
    steps: transient inputs, literal and prefix extraction, a grid with gated-out
    and duplicate rows."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2510_08288_b200.sharded import (robust_rg_parallel_sharded,
                                               robust_rg_sequential_sharded)

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29534")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        m = rg.DisturbanceModel.scaled(0.02, 3)
        box = rg.ConstraintSet(-0.9, 0.9)
        cases = [(0.4, 2.2, False, 32), (0.4, 2.2, True, 32), (1.2, -2.5, False, 32),
                 (0.9, 0.9, False, 16), (0.0, 2.5, True, 9)]
        for i, (vp, r, prefix, M) in enumerate(cases):
            cfg = rg.GovernorConfig(j_star=128, n_sim=3000, m_grid=M, prefix_mode=prefix)
            scen = rg.sample_scenarios(m, 3000, 129, seed=70 + i)
            x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + 0.02
            a = rg.robust_rg_parallel(PLANT, x0, rg.GovernorState(vp), r, box, scen, cfg)
            b = robust_rg_parallel_sharded(PLANT, x0, rg.GovernorState(vp), r, box, scen, cfg)
            assert (a.kappa_opt, a.feasible, a.v_applied) == (b.kappa_opt, b.feasible,
                                                              b.v_applied), (i, a, b)
            c = rg.robust_rg_sequential(PLANT, x0, rg.GovernorState(vp), r, box, scen, cfg)
            d = robust_rg_sequential_sharded(PLANT, x0, rg.GovernorState(vp), r, box, scen,
                                             cfg)
            assert (c.kappa_opt, c.feasible, c.v_applied) == (d.kappa_opt, d.feasible,
                                                              d.v_applied), (i, c, d)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1, 31, 33, 1000, 148 * 32 + 1, 10_000, 100_000])
@pytest.mark.parametrize("mode", ["fused", "staged"])
def test_persistent_joint_equals_per_iteration_launches(n, mode):
    """The persistent speculative kernel (a tree of 1, 3 or 7 candidates per round, grid
    barrier, every block walking the same decisions) against the one-kernel-per-iteration
    form: same kappa, found and rollout count on transient-binding inputs (where verdicts
    flip along the path), and the same as the exact Alg. 2.  100k scenarios exceed one
    wave and take the per-iteration launches in both calls."""
    ctx = _capi.context(0)
    rng = np.random.default_rng(n)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
    lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
    for trial in range(6):
        j_star = (128, 256, 7)[trial % 3]
        n_kappa = (8, 1, 20)[trial % 3]
        prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, j_star, 0)
        vp = float(rng.uniform(-1, 1))
        r = float(rng.uniform(-2.5, 2.5))
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.05, 0.05, 3)
        sc = _capi.make_scenarios(7000 + trial, 3, n, m.lo, m.span)
        per = ctx.bisect_joint(prob, x0, vp, r, n_kappa, None, n, sc, rng_mode=mode,
                               per_iteration=True)
        one = ctx.bisect_joint(prob, x0, vp, r, n_kappa, None, n, sc, rng_mode=mode)
        assert (one.kappa, one.found, one.cells) == (per.kappa, per.found, per.cells), trial
        a2, _, _ = ctx.bisect(prob, x0, vp, r, n_kappa, None, n, sc, rng_mode=mode)
        assert (one.kappa, one.found) == (a2.kappa, a2.found), trial


def test_persistent_joint_repeated_calls_and_long_searches():
    """Back-to-back searches reuse the per-round words and the barrier (reset by the last
    block out); n_kappa = 63 is the persistent kernel's limit, 64 falls back to one launch
    per iteration.  Results stay those of the per-iteration form."""
    ctx = _capi.context(0)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
    lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
    prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 64, 0)
    x0 = np.array([0.2, 0.4, 0.1])
    for rep in range(40):
        nk = (63, 64, 8, 30)[rep % 4]
        sc = _capi.make_scenarios(100 + rep % 5, 0, 5000, m.lo, m.span)
        a = ctx.bisect_joint(prob, x0, 0.4, 2.2 - 0.1 * (rep % 7), nk, None, 5000, sc)
        b = ctx.bisect_joint(prob, x0, 0.4, 2.2 - 0.1 * (rep % 7), nk, None, 5000, sc,
                             per_iteration=True)
        assert (a.kappa, a.found, a.cells) == (b.kappa, b.found, b.cells), rep


def test_persistent_joint_dense_and_nominal_sources(golden, orc):
    """Dense host scenarios (staged from the caller's tensor) and a single scenario."""
    ctx = _capi.context(0)
    for idx in range(N_BIS):
        c = bis_case(golden, idx)
        if c["n_kappa"] + 1 > 64:
            continue
        dist = orc.sample(c["seed"], c["n_sim"], c["j_star"] + 1, c["ranges"])
        tight = rg.tighten(_cset(c), c["eps"])
        lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
        prob = _capi.Problem(0.01, c["lower"], c["upper"], lo, hi, c["j_star"], 0)
        one = ctx.bisect_joint(prob, c["x0"], c["v_prev"], c["r"], c["n_kappa"], dist,
                               c["n_sim"], None)
        per = ctx.bisect_joint(prob, c["x0"], c["v_prev"], c["r"], c["n_kappa"], dist,
                               c["n_sim"], None, per_iteration=True)
        assert (one.kappa, one.found, one.cells) == (per.kappa, per.found, per.cells), c["name"]
        d1 = dist[:1]
        one = ctx.bisect_joint(prob, c["x0"], c["v_prev"], c["r"], c["n_kappa"], d1, 1, None)
        per = ctx.bisect_joint(prob, c["x0"], c["v_prev"], c["r"], c["n_kappa"], d1, 1, None,
                               per_iteration=True)
        assert (one.kappa, one.found, one.cells) == (per.kappa, per.found, per.cells), c["name"]


def test_speculative_search_stress_against_per_iteration():
    """200 random transient-binding searches at sizes where the speculation tree has 7,
    3 and 1 candidates per round (n = 300, 2000, 4000): kappa / found / rollout count
    equal the one-candidate-per-iteration search's."""
    ctx = _capi.context(0)
    rng = np.random.default_rng(2026)
    for trial in range(200):
        n = (300, 2000, 4000)[trial % 3]
        mag = float(rng.choice([0.001, 0.02, 0.05]))
        m = rg.DisturbanceModel.scaled(mag, 3)
        eps = float(rng.choice([0.05, 0.2]))
        tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), eps)
        lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
        j_star = int(rng.choice([16, 64, 200]))
        prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, j_star, 0)
        vp = float(rng.uniform(-1.2, 1.2))
        r = float(rng.uniform(-3, 3))
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.08, 0.08, 3)
        sc = _capi.make_scenarios(int(rng.integers(0, 2**62)), 0, n, m.lo, m.span)
        nk = int(rng.choice([4, 8, 12]))
        one = ctx.bisect_joint(prob, x0, vp, r, nk, None, n, sc)
        per = ctx.bisect_joint(prob, x0, vp, r, nk, None, n, sc, per_iteration=True)
        assert (one.kappa, one.found, one.cells) == (per.kappa, per.found, per.cells), trial
