"""Parity of the CUDA path with the reference (golden fixtures) and the CPU oracle.

Everything here runs through the C ABI on a B200 (``-m gpu``).  The bar is
bit-exact: identical cell statuses and step counts, identical feasibility
matrices, identical bisection paths, identical kappa and v_t doubles.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
from paper_2510_08288_b200.governor import bisect_paths
from conftest import GOLDEN, bis_case, fill_case

pytestmark = pytest.mark.gpu

with np.load(GOLDEN) as _z:
    N_FILL = len(_z["fill_names"])
    N_BIS = len(_z["bis_names"])

MASK = (1 << 64) - 1
PLANT = rg.make_plant("surrogate-fc")


@pytest.fixture(scope="module")
def ctx():
    return _capi.context(0)


def _cset(c):
    return rg.ConstraintSet(c["lower"], c["upper"], c["anchor"])


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


# ----------------------------------------------------------------- tanh

def test_device_tanh_matches_host_libm_golden(ctx, golden, orc):
    x = golden["tanh_x"]
    y = ctx.tanh(x)
    assert np.array_equal(_bits(y), _bits(orc.libm_tanh(x)))
    # the fixture was written on the build container's libm (FMA build)
    if ctx.tanh_variant == _capi.RG_TANH_FMA:
        assert np.array_equal(_bits(y), _bits(golden["tanh_libm"]))


def test_device_tanh_bit_exact_sweep(ctx, orc):
    rng = np.random.default_rng(5)
    x = np.concatenate([
        rng.uniform(-3, 3, 2_000_000), rng.uniform(-25, 25, 500_000),
        np.ldexp(rng.uniform(0.5, 1.0, 200_000), rng.integers(-64, 6, 200_000)),
        -np.ldexp(rng.uniform(0.5, 1.0, 200_000), rng.integers(-64, 6, 200_000)),
        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 22.0, -22.0, 5e-324, 1.0, -1.0]),
    ])
    y = ctx.tanh(x)
    ref = orc.libm_tanh(x)
    mism = np.flatnonzero(_bits(y) != _bits(ref))
    assert mism.size == 0, f"{mism.size} mismatches, first x={x[mism[:5]]}"


# ----------------------------------------------------------------- RNG

def test_sample_scenarios_bit_exact(golden):
    model = rg.DisturbanceModel(ranges=((-0.003, 0.001), (0.0, 0.002), (-1e-4, 1e-4)))
    s = rg.sample_scenarios(model, 5, 9, seed=2**63 + 5)
    assert np.array_equal(s.data, golden["scen_small"])
    big = rg.sample_scenarios(rg.DisturbanceModel.scaled(0.001, 3), 1000, 257, seed=7)
    assert hashlib.sha256(big.data.tobytes()).digest() == golden["scen_big_sha"].tobytes()
    wrap = rg.sample_scenarios(rg.DisturbanceModel.scaled(0.001, 3), 3, 5,
                               seed=((MASK - 1) + 5) & MASK)
    assert np.array_equal(wrap.data, golden["scen_wrap"])
    unit = rg.DisturbanceModel(ranges=((0.0, 1.0),) * 3)
    k0set = rg.ScenarioSet.generated(unit, 4, 6, 2**64 - 3, k0=1_000_000)
    assert np.array_equal(k0set.data, golden["scen_small_k0"])


def test_sample_prefix_and_shards(orc):
    model = rg.DisturbanceModel.scaled(1.0, 3)
    big = rg.sample_scenarios(model, 300, 17, seed=42)
    assert np.array_equal(big.prefix(16).data, big.data[:16])
    parts = np.concatenate([big.shard(r, 3).data for r in range(3)])
    assert np.array_equal(parts, big.data)
    assert np.array_equal(big.data, orc.sample(42, 300, 17, model.ranges))


# ----------------------------------------------------------------- cells

def _problem(c, tight=None):
    cset = _cset(c)
    tight = tight or rg.tighten(cset, c["eps"])
    lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
    return _capi.Problem(0.01, cset.lower, cset.upper, lo, hi, c["j_star"], 0)


@pytest.mark.parametrize("source", ["staged", "rng"])
@pytest.mark.parametrize("idx", range(N_FILL))
def test_fill_cells_bit_exact(ctx, golden, idx, source):
    c = fill_case(golden, idx)
    grid = rg.grid_kappas(c["m_grid"])
    v_rows = np.array([rg.update_setpoint(c["v_prev"], c["r"], float(k)) for k in grid])
    S = np.full((c["m_grid"], c["n_sim"]), 7, np.uint8)
    steps = np.full((c["m_grid"], c["n_sim"]), -1, np.int32)
    rows = np.arange(c["m_grid"], dtype=np.int32)
    if source == "staged":
        dist = rg.sample_scenarios(rg.DisturbanceModel(c["ranges"]), c["n_sim"],
                                   c["j_star"] + 1, c["seed"]).data
        ctx.fill(_problem(c), c["x0"], v_rows, rows, dist, c["n_sim"], None, S, steps)
    else:
        m = rg.DisturbanceModel(c["ranges"])
        scen = _capi.make_scenarios(c["seed"], 0, c["n_sim"], m.lo, m.span)
        ctx.fill(_problem(c), c["x0"], v_rows, rows, None, c["n_sim"], scen, S, steps)
    assert np.array_equal(S, c["S_all"]), c["name"]
    assert np.array_equal(steps, c["steps_all"]), c["name"]


@pytest.mark.parametrize("idx", range(N_FILL))
def test_fill_feasibility_matches_reference(golden, idx):
    c = fill_case(golden, idx)
    scen = rg.sample_scenarios(rg.DisturbanceModel(c["ranges"]), c["n_sim"], c["j_star"] + 1,
                               c["seed"])
    for s in (scen, rg.ScenarioSet(scen.data)):   # generated and dense inputs
        stats = {}
        P = rg.fill_feasibility("cuda", PLANT, c["x0"], c["v_prev"], c["r"],
                                rg.grid_kappas(c["m_grid"]), s, _cset(c), c["eps"],
                                c["j_star"], stats=stats)
        assert np.array_equal(P, c["P"]), c["name"]
        got = [stats[k] for k in ("sims_run", "early_terms", "overflows", "ss_pruned_rows",
                                  "dedup_rows")]
        assert got == [int(v) for v in c["stats"]], c["name"]


@pytest.mark.parametrize("keep", [True, False])
@pytest.mark.parametrize("idx", range(N_FILL))
def test_robust_rg_parallel_matches_reference(golden, idx, keep):
    c = fill_case(golden, idx)
    cfg = rg.GovernorConfig(j_star=c["j_star"], epsilon=c["eps"], m_grid=c["m_grid"],
                            n_sim=c["n_sim"], prefix_mode=c["prefix"], keep_matrix=keep)
    scen = rg.sample_scenarios(rg.DisturbanceModel(c["ranges"]), c["n_sim"], c["j_star"] + 1,
                               c["seed"])
    for s in (scen, rg.ScenarioSet(scen.data)):
        state = rg.GovernorState(c["v_prev"])
        res = rg.robust_rg_parallel(PLANT, c["x0"], state, c["r"], _cset(c), s, cfg)
        assert (res.kappa_opt, res.v_applied, float(res.feasible)) == \
            tuple(float(v) for v in c["result"]), c["name"]
        if keep:
            assert np.array_equal(res.matrix, c["P"]), c["name"]
            d = res.diagnostics
            got = [d[k] for k in ("sims_run", "early_terms", "overflows", "ss_pruned_rows",
                                  "dedup_rows")]
            assert got == [int(v) for v in c["stats"]], c["name"]


# ----------------------------------------------------------------- bisection

@pytest.mark.parametrize("idx", range(N_BIS))
def test_robust_rg_sequential_matches_reference(golden, idx):
    c = bis_case(golden, idx)
    cfg = rg.GovernorConfig(j_star=c["j_star"], epsilon=c["eps"], n_kappa=c["n_kappa"],
                            n_sim=c["n_sim"])
    scen = rg.sample_scenarios(rg.DisturbanceModel(c["ranges"]), c["n_sim"], c["j_star"] + 1,
                               c["seed"])
    for s in (scen, rg.ScenarioSet(scen.data)):
        res = rg.robust_rg_sequential(PLANT, c["x0"], rg.GovernorState(c["v_prev"]), c["r"],
                                      _cset(c), s, cfg)
        d = res.diagnostics
        assert (res.kappa_opt, res.v_applied, float(res.feasible), d["sims_run"],
                d["early_terms"]) == tuple(float(v) for v in c["result"]), c["name"]
    kap, fnd, cel, erl, pk, po = bisect_paths(PLANT, c["x0"], c["v_prev"], c["r"], _cset(c),
                                              scen, cfg)
    per = np.stack([kap, fnd, cel, erl], axis=1).astype(np.float64)
    assert np.array_equal(per, c["per"]), c["name"]
    ref_k, ref_ok = c["paths"][..., 0], c["paths"][..., 1]
    used = ~np.isnan(ref_k)
    assert np.array_equal(np.isnan(pk), ~used)
    assert np.array_equal(pk[used], ref_k[used])
    assert np.array_equal(po[used], ref_ok[used].astype(np.uint8))


def test_nominal_bisection_anchor(golden):
    res = rg.bisection_rg(PLANT, np.zeros(3), rg.GovernorState(0.0), 2.5,
                          rg.ConstraintSet(-0.9, 0.9), rg.GovernorConfig())
    d = res.diagnostics
    assert (res.kappa_opt, res.v_applied, float(res.feasible), d["sims_run"],
            d["early_terms"]) == tuple(float(v) for v in golden["nominal_anchor"])
    assert res.kappa_opt == 0.5078125


def test_closed_loop_c1_bisection_trace(golden):
    """Config 1: desk-scale nominal bisection governor, 2000 steps, v_t bit-exact."""
    from paper_2510_08288_b200.harness import run_closed_loop_bisection

    prof = golden["desk_profile"]
    rows = run_closed_loop_bisection(PLANT, rg.ConstraintSet(-0.9, 0.9),
                                     rg.DisturbanceModel.scaled(0.001, 3), rg.GovernorConfig(),
                                     prof, 2000, 2024)
    ref = golden["c1_trace"]
    got = np.array([[r.kappa_opt, r.v_applied, float(r.feasible), y, r.diagnostics["sims_run"],
                     r.diagnostics["early_terms"]] for r, y in rows])
    assert np.array_equal(got, ref)


def test_closed_loop_desk_grid_trace(golden):
    from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop

    prof = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
    rec = run_closed_loop(PLANT, rg.ConstraintSet(-0.9, 0.9),
                          rg.DisturbanceModel.scaled(0.001, 3),
                          rg.GovernorConfig(n_sim=64), prof, 2000, 2024)
    assert not rec.aborted
    got = np.array([[row[2], row[3], row[4], float(row[5])] for row in rec.rows])
    assert np.array_equal(got, golden["desk_grid_trace"])


def test_closed_loop_c3_truncated(golden):
    from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop

    prof = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
    rec = run_closed_loop(PLANT, rg.ConstraintSet(-0.9, 0.9),
                          rg.DisturbanceModel.scaled(0.001, 3),
                          rg.GovernorConfig(n_sim=1000), prof, 40, 2024)
    got = np.array([[row[2], row[3], row[4], float(row[5])] for row in rec.rows])
    assert np.array_equal(got, golden["c3_trace40"])


@pytest.mark.parametrize("case", ["lit", "prefix"])
@pytest.mark.parametrize("device_loop", [1, 0])
def test_closed_loop_transient_golden(case, device_loop):
    """Closed loops with transients against the real reference (tests/golden/
    make_loop_transient_golden.py): references jumping every 60 steps under larger
    disturbances, so up to every row is live (literal mode: 2.6 live rows per step on
    average at 2000 scenarios, up to 32; prefix mode at M = 16).  The rows (v, y, kappa,
    feasible) and the diagnostics (sims_run, early_terms) equal the reference's every step,
    through the device loop (k_loop_ts, several time-split passes per step) and through one
    grid-step launch per step."""
    from paper_2510_08288_b200 import _capi
    from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop

    with np.load(GOLDEN.with_name("loop_transient.npz")) as z:
        g = {k: z[k] for k in z.files}
    c = lambda k: g[f"{case}_{k}"].item()
    cfg = rg.GovernorConfig(j_star=c("j_star"), m_grid=c("m_grid"), n_sim=c("n_sim"),
                            prefix_mode=bool(c("prefix_mode")))
    prof = ReferenceProfile(tuple((int(t), float(r)) for t, r in g["profile"]))
    ctx = _capi.context(0)
    ctx.set_option("no_device_loop", 1 - device_loop)
    try:
        rec = run_closed_loop(PLANT, rg.ConstraintSet(-0.9, 0.9, anchor=0.0),
                              rg.DisturbanceModel.scaled(c("scale"), 3), cfg, prof,
                              int(g["steps"]), c("seed"))
        assert ctx.get_option("last_loop_device") == device_loop
    finally:
        ctx.set_option("no_device_loop", 0)
    assert not rec.aborted
    got = np.array([[row[2], row[3], row[4], float(row[5])] for row in rec.rows])
    diag = np.array([[int(d.split(",")[4]), int(d.split(",")[5])] for d in rec.diag_rows])
    assert np.array_equal(got, g[f"{case}_trace"])
    assert np.array_equal(diag, g[f"{case}_diag"])


def test_closed_loop_c3_10k_full_trace():
    """C3 at its named size: 10,000 scenarios per step, the whole 2000-step desk trace
    (rise to r = 0.4, r = 2.5 at t = 400, r = -2.5 at t = 1000, r = 0.2 at t = 1600;
    1200 steps with kappa < 1), equal bit for bit to the real reference's trace
    (tests/golden/make_c3_golden.py, multicore fill in the build container)."""
    from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop

    with np.load(GOLDEN.with_name("c3_10k_trace.npz")) as z:
        want, steps, n_sim, seed = z["trace"], int(z["steps"]), int(z["n_sim"]), int(z["seed"])
    prof = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
    rec = run_closed_loop(PLANT, rg.ConstraintSet(-0.9, 0.9),
                          rg.DisturbanceModel.scaled(0.001, 3),
                          rg.GovernorConfig(n_sim=n_sim), prof, steps, seed)
    assert not rec.aborted
    got = np.array([[row[2], row[3], row[4], float(row[5])] for row in rec.rows])
    assert np.array_equal(got, want)


def test_closed_loop_c5_batch_10k():
    """C5's batched path at 10k scenarios per episode: episode seeds base + e, one
    rg_grid_step_batch launch per step, the whole 2000-step trace.  Episode 0 (seed 2024)
    equals the real reference's C3 trace; the others equal their single-episode loops."""
    from paper_2510_08288_b200.harness import (ReferenceProfile, run_closed_loop,
                                               run_closed_loop_batch)

    with np.load(GOLDEN.with_name("c3_10k_trace.npz")) as z:
        want, steps, n_sim, seed = z["trace"], int(z["steps"]), int(z["n_sim"]), int(z["seed"])
    prof = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
    box, model = rg.ConstraintSet(-0.9, 0.9), rg.DisturbanceModel.scaled(0.001, 3)
    cfg = rg.GovernorConfig(n_sim=n_sim)
    seeds = [seed + e for e in range(4)]
    recs = run_closed_loop_batch(PLANT, box, model, cfg, prof, steps, seeds)
    got = np.array([[row[2], row[3], row[4], float(row[5])] for row in recs[0].rows])
    assert np.array_equal(got, want)
    for e in (1, 3):
        single = run_closed_loop(PLANT, box, model, cfg, prof, steps, seeds[e])
        assert [row[:6] for row in recs[e].rows] == [row[:6] for row in single.rows]


# ----------------------------------------------------------------- edges & errors

def test_errors_map_to_reference_types():
    box = rg.ConstraintSet(-0.9, 0.9)
    cfg = rg.GovernorConfig(j_star=64, n_sim=1)
    with pytest.raises(rg.ConfigError):   # short horizon (governor.py:175-178)
        rg.robust_rg_parallel(PLANT, np.zeros(3), rg.GovernorState(), 1.0, box,
                              rg.zero_scenarios(3, 64), cfg)
    with pytest.raises(rg.ConfigError):   # non-finite state
        rg.robust_rg_parallel(PLANT, np.array([np.nan, 0, 0]), rg.GovernorState(), 1.0, box,
                              rg.zero_scenarios(3, 65), cfg)
    class OtherPlant(rg.Plant):   # neither the surrogate nor a linear plant
        kernel_kind = None
        state_dim = 1
    with pytest.raises(rg.BackendUnavailableError):  # backend_gpu.py:66-71
        rg.fill_feasibility("cuda", OtherPlant(), np.zeros(1), 0.0, 1.0, rg.grid_kappas(4),
                            rg.ScenarioSet(np.zeros((1, 33, 1))), box, 0.05, 32)
    with pytest.raises(rg.ConfigError):
        rg.fill_feasibility("serial", PLANT, np.zeros(3), 0.0, 1.0, rg.grid_kappas(4),
                            rg.zero_scenarios(3, 33), box, 0.05, 32)
    with pytest.raises(rg.ConfigError):
        rg.robust_rg_sequential(PLANT, np.zeros(3), rg.GovernorState(), 1.0, box,
                                rg.zero_scenarios(3, 33), rg.GovernorConfig(j_star=32, n_sim=4))


def test_infeasible_policies():
    box = rg.ConstraintSet(-0.9, 0.9)
    x_bad = np.array([2.0, 0.0, 0.0])
    cfg = rg.GovernorConfig(j_star=32, n_sim=1, m_grid=8)
    state = rg.GovernorState(0.7)
    res = rg.robust_rg_parallel(PLANT, x_bad, state, 1.0, box, rg.zero_scenarios(3, 33), cfg)
    assert (res.kappa_opt, res.v_applied, res.feasible, state.v_prev) == (0.0, 0.7, False, 0.7)
    with pytest.raises(rg.InfeasibleError):
        rg.robust_rg_parallel(PLANT, x_bad, rg.GovernorState(0.7), 1.0, box,
                              rg.zero_scenarios(3, 33),
                              rg.GovernorConfig(j_star=32, n_sim=1, m_grid=8,
                                                infeasible_policy="error"))


def test_repeated_steps_reset_device_accumulators():
    """The last-block reset must leave the counters clean for the next launch."""
    box = rg.ConstraintSet(-0.9, 0.9)
    cfg = rg.GovernorConfig(j_star=128, n_sim=500, m_grid=32)
    model = rg.DisturbanceModel.scaled(0.02, 3)
    outs = []
    for rep in range(3):
        for r in (2.5, 0.3):
            scen = rg.sample_scenarios(model, 500, 129, seed=11)
            res = rg.robust_rg_parallel(PLANT, np.zeros(3), rg.GovernorState(0.0), r, box,
                                        scen, cfg)
            outs.append((r, res.kappa_opt, res.diagnostics["early_terms"]))
    assert outs[0:2] == outs[2:4] == outs[4:6]


def test_c4_million_scenario_step_matches_reference():
    """C4 at its full per-step size: the robust grid step over 2^20 scenarios, j* = 256,
    through the public API.  The 32 x 2^20 matrix P (packed-bit sha256 and per-row
    counts) and (kappa, v, feasible) equal the real reference's
    (tests/golden/make_c4_golden.py, multicore fill on the build container)."""
    with np.load(GOLDEN.with_name("c4_1m_step.npz")) as z:
        g = {k: z[k] for k in z.files}
    n, j_star, m = int(g["n_sim"]), int(g["j_star"]), int(g["m_grid"])
    v_prev, r = float(g["v_prev"]), float(g["r"])
    scen = rg.sample_scenarios(rg.DisturbanceModel.scaled(float(g["range"]), 3), n, j_star + 1,
                               seed=int(g["seed"]))
    state = rg.GovernorState(v_prev)
    res = rg.robust_rg_parallel(PLANT, g["x0"], state, r, rg.ConstraintSet(-0.9, 0.9, 0.0), scen,
                                rg.GovernorConfig(j_star=j_star, m_grid=m, n_sim=n))
    P = res.matrix
    assert P.shape == (m, n)
    assert np.array_equal(P.sum(axis=1), g["row_counts"])
    assert hashlib.sha256(np.packbits(P, axis=1).tobytes()).digest() == g["p_sha"].tobytes()
    assert (res.kappa_opt, res.v_applied, float(res.feasible)) == tuple(g["result"])


def test_c4_million_scenario_alg2_matches_reference():
    """Alg. 2 (robust_rg_sequential) over the same 2^20 scenarios: kappa, v, feasible
    and the rollout/early-termination counters equal the real reference's
    (tests/golden/make_c4_seq_golden.py); the joint search lands on the same kappa."""
    with np.load(GOLDEN.with_name("c4_1m_step.npz")) as z:
        g = {k: z[k] for k in z.files}
    with np.load(GOLDEN.with_name("c4_1m_seq.npz")) as z:
        want = tuple(float(v) for v in z["result"])
    n, j_star = int(g["n_sim"]), int(g["j_star"])
    v_prev, r = float(g["v_prev"]), float(g["r"])
    scen = rg.sample_scenarios(rg.DisturbanceModel.scaled(float(g["range"]), 3), n, j_star + 1,
                               seed=int(g["seed"]))
    box = rg.ConstraintSet(-0.9, 0.9, 0.0)
    cfg = rg.GovernorConfig(j_star=j_star, n_sim=n, n_kappa=8)
    res = rg.robust_rg_sequential(PLANT, g["x0"], rg.GovernorState(v_prev), r, box, scen, cfg)
    d = res.diagnostics
    assert (res.kappa_opt, res.v_applied, float(res.feasible), d["sims_run"],
            d["early_terms"]) == want
    jt = rg.robust_rg_joint(PLANT, g["x0"], rg.GovernorState(v_prev), r, box, scen, cfg)
    assert (jt.kappa_opt, jt.feasible) == (res.kappa_opt, res.feasible)


# ----------------------------------------------------------------- C2 transient variant

def _c2_transient():
    with np.load(GOLDEN.with_name("c2_transient.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("source", ["generated", "dense"])
@pytest.mark.parametrize("trial", range(16))
def test_c2_transient_grid_alg2_joint_match_reference(trial, source):
    """C2's transient-binding variant at its named size (1000 scenarios, j* = 256, M = 32,
    scaled(0.02), state off equilibrium; tests/golden/make_c2_transient_golden.py): the
    device grid step's P, decision and stats, Alg. 2's five numbers and the joint search's
    kappa / feasible equal the real reference's -- through the public API, with the
    scenarios generated on the device or passed as a dense host tensor."""
    g = _c2_transient()
    n, js, m, nk = int(g["n_sim"]), int(g["j_star"]), int(g["m_grid"]), int(g["n_kappa"])
    x0, vp, r = g["x0"][trial], float(g["v_prev"][trial]), float(g["r"][trial])
    scen = rg.sample_scenarios(rg.DisturbanceModel.scaled(float(g["range"]), 3), n, js + 1,
                               seed=int(g["seed"][trial]))
    if source == "dense":
        scen = rg.ScenarioSet(scen.data)
    box = rg.ConstraintSet(-0.9, 0.9, 0.0)
    cfg = rg.GovernorConfig(j_star=js, m_grid=m, n_sim=n, n_kappa=nk)
    res = rg.robust_rg_parallel(PLANT, x0, rg.GovernorState(vp), r, box, scen, cfg)
    assert np.array_equal(np.packbits(res.matrix, axis=1), g["p_packed"][trial])
    assert [res.kappa_opt, res.v_applied, float(res.feasible)] == g["grid"][trial].tolist()
    d = res.diagnostics
    assert [d["sims_run"], d["early_terms"], d["overflows"], d["ss_pruned_rows"],
            d["dedup_rows"]] == g["stats"][trial].tolist()
    seq = rg.robust_rg_sequential(PLANT, x0, rg.GovernorState(vp), r, box, scen, cfg)
    assert [seq.kappa_opt, seq.v_applied, float(seq.feasible), seq.diagnostics["sims_run"],
            seq.diagnostics["early_terms"]] == g["seq"][trial].tolist()
    jt = rg.robust_rg_joint(PLANT, x0, rg.GovernorState(vp), r, box, scen, cfg)
    assert (jt.kappa_opt, float(jt.feasible)) == (seq.kappa_opt, float(seq.feasible))
    assert jt.v_applied == seq.v_applied
