"""Batched episodes (BASELINE C5): the batched device step and closed loop must
equal the single-episode paths, and the vectorised true-plant step must equal
the reference's scalar rk4_step (numpy's vector and scalar tanh agree)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2510_08288_b200 as rg
from paper_2510_08288_b200.harness import (ReferenceProfile, _rk4_batch, run_closed_loop,
                                           run_closed_loop_batch)

PLANT = rg.make_plant("surrogate-fc")
BOX = rg.ConstraintSet(-0.9, 0.9)
PROFILE = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))


def test_rk4_batch_equals_scalar_step():
    rng = np.random.default_rng(0)
    X = np.concatenate([rng.uniform(-1, 1, (3000, 3)), rng.uniform(-30, 30, (1000, 3))])
    V = rng.uniform(-3, 3, X.shape[0])
    got = _rk4_batch(0.01, X, V)
    ref = np.stack([PLANT.step(X[i], float(V[i])) for i in range(X.shape[0])])
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


def test_numpy_tanh_vector_equals_scalar():
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.uniform(-3, 3, 200_000), rng.uniform(-25, 25, 50_000)])
    sc = np.array([np.tanh(np.float64(v)) for v in x])
    assert np.array_equal(np.tanh(x).view(np.uint64), sc.view(np.uint64))


@pytest.mark.gpu
def test_batch_step_equals_single_steps():
    rng = np.random.default_rng(7)
    E, n = 24, 300
    model = rg.DisturbanceModel.scaled(0.02, 3)
    cfg = rg.GovernorConfig(j_star=128, m_grid=32, n_sim=n)
    vp = rng.uniform(-1, 1, E)
    r = rng.uniform(-2.5, 2.5, E)
    X = np.stack([[np.tanh(v), v, np.tanh(v) / 2] for v in vp]) + rng.uniform(-0.05, 0.05, (E, 3))
    X[3] = [2.0, 0.0, 0.0]          # infeasible episode (holds)
    r[5] = vp[5]                    # all rows duplicate
    seeds = [int(s) for s in rng.integers(0, 2**63, E)] + []
    seeds[2] = 2**64 - 3
    kap, v, feas, _ = rg.robust_rg_parallel_batch(PLANT, X, vp, r, BOX, model, n, seeds, cfg)
    for e in range(E):
        scen = rg.sample_scenarios(model, n, cfg.j_star + 1, seed=seeds[e])
        res = rg.robust_rg_parallel(PLANT, X[e], rg.GovernorState(float(vp[e])), float(r[e]),
                                    BOX, scen, cfg)
        assert (kap[e], v[e], bool(feas[e])) == (res.kappa_opt, res.v_applied, res.feasible), e


@pytest.mark.gpu
def test_closed_loop_batch_equals_single_episode_loops(golden):
    model = rg.DisturbanceModel.scaled(0.001, 3)
    cfg = rg.GovernorConfig(n_sim=64)
    seeds = [2024, 3001, 3002, 77]
    recs = run_closed_loop_batch(PLANT, BOX, model, cfg, PROFILE, 2000, seeds)
    got = np.array([[row[2], row[3], row[4], float(row[5])] for row in recs[0].rows])
    assert np.array_equal(got, golden["desk_grid_trace"])   # the reference's own trace
    for e in (1, 3):
        single = run_closed_loop(PLANT, BOX, model, cfg, PROFILE, 600, seeds[e])
        assert [row[:6] for row in recs[e].rows[:600]] == [row[:6] for row in single.rows]


def test_parse_nsim_spec_and_csv(tmp_path):
    from paper_2510_08288_b200.harness import (RunRecord, TimingRecord, emit_csv,
                                               parse_nsim_spec)

    assert parse_nsim_spec("1:4:1,32:96:32") == [1, 2, 3, 4, 32, 64, 96]
    assert parse_nsim_spec("64, 128") == [64, 128]
    with pytest.raises(rg.ConfigError):
        parse_nsim_spec("5:1:1")
    emit_csv([TimingRecord("cuda", 64, 32, 3, "kernel-only", 2.0, 1.0, 3.0)], tmp_path / "t.csv")
    assert (tmp_path / "t.csv").read_text().splitlines() == [
        "backend,n_sim,mode,mean_us,min_us,max_us,reps", "cuda,64,kernel-only,2.0,1.0,3.0,3"]
    emit_csv(RunRecord(rows=[(0, 0.4, 0.4, 0.0, 1.0, True, 12)], config={}, seed=1),
             tmp_path / "r.csv")
    assert (tmp_path / "r.csv").read_text().splitlines()[1] == "0,0.4,0.4,0.0,1.0,1,12"


@pytest.mark.gpu
def test_bench_sweep_on_device():
    from paper_2510_08288_b200.harness import bench_sweep

    recs = bench_sweep(PLANT, BOX, rg.DisturbanceModel.scaled(0.001, 3),
                       rg.GovernorConfig(j_star=64), [64, 256], ["cuda", "serial"], reps=3)
    assert [(r.backend, r.n_sim, r.mode, r.skipped) for r in recs] == [
        ("cuda", 64, "kernel-only", False), ("cuda", 64, "end-to-end", False),
        ("cuda", 256, "kernel-only", False), ("cuda", 256, "end-to-end", False),
        ("serial", 64, "kernel-only", True), ("serial", 64, "end-to-end", True),
        ("serial", 256, "kernel-only", True), ("serial", 256, "end-to-end", True)]
    assert all(r.min_us > 0 for r in recs if not r.skipped)


@pytest.mark.gpu
def test_closed_loop_batch_over_devices_equals_one_device():
    """C5's N-device form: episodes split over devices (contiguous ranges, concurrent
    calls from host threads).  On the one-GPU box the 'devices' are the same GPU listed
    three times -- the split, the concurrent calls on one context and the merge are the
    code that runs on 8 GPUs.  Every episode equals the one-device batch and, for two
    episodes, the single-episode loop."""
    model = rg.DisturbanceModel.scaled(0.001, 3)
    cfg = rg.GovernorConfig(n_sim=300)
    seeds = [2024 + e for e in range(10)]
    one = run_closed_loop_batch(PLANT, BOX, model, cfg, PROFILE, 700, seeds)
    many = run_closed_loop_batch(PLANT, BOX, model, cfg, PROFILE, 700, seeds, devices=[0, 0, 0])
    for a, b in zip(one, many):
        assert [row[:6] for row in a.rows] == [row[:6] for row in b.rows]
    for e in (0, 9):
        single = run_closed_loop(PLANT, BOX, model, cfg, PROFILE, 700, seeds[e])
        assert [row[:6] for row in many[e].rows] == [row[:6] for row in single.rows]


@pytest.mark.gpu
def test_batch_step_infeasible_policy_error():
    """robust_rg_parallel_batch honours infeasible_policy="error" like the single call
    (governor.py:562-573): an episode with no feasible candidate raises InfeasibleError."""
    model = rg.DisturbanceModel.scaled(0.02, 3)
    X = np.array([[0.0, 0.0, 0.0], [2.0, 0.0, 0.0]])   # episode 1 starts outside the set
    for policy, raises in (("hold", False), ("error", True)):
        cfg = rg.GovernorConfig(j_star=64, m_grid=8, n_sim=50, infeasible_policy=policy)
        if raises:
            with pytest.raises(rg.InfeasibleError):
                rg.robust_rg_parallel_batch(PLANT, X, np.zeros(2), np.full(2, 0.5), BOX, model,
                                            50, [1, 2], cfg)
        else:
            kap, v, feas, _ = rg.robust_rg_parallel_batch(PLANT, X, np.zeros(2), np.full(2, 0.5),
                                                          BOX, model, 50, [1, 2], cfg)
            assert feas.tolist() == [True, False] and v[1] == 0.0


@pytest.mark.gpu
def test_c5_named_size_batch_equals_single_episode_loops():
    """C5 at its named size for three closed-loop steps: 4096 episodes x 10k scenarios in one
    batched launch per step (131k candidate rows at t = 0, ~643k blocks of the pairs kernel,
    the staged chunks of the t = 0 step).  Sampled episodes equal their single-episode loops."""
    model = rg.DisturbanceModel.scaled(0.001, 3)
    cfg = rg.GovernorConfig(n_sim=10_000)
    seeds = [2024 + e for e in range(4096)]
    recs = run_closed_loop_batch(PLANT, BOX, model, cfg, PROFILE, 3, seeds)
    assert len(recs) == 4096 and all(len(r.rows) == 3 for r in recs)
    for e in (0, 1, 1000, 2047, 4095):
        single = run_closed_loop(PLANT, BOX, model, cfg, PROFILE, 3, seeds[e])
        assert [row[:6] for row in recs[e].rows] == [row[:6] for row in single.rows], e
