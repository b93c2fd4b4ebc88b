"""Kernel-level parity on the B200: the lockstep tanh, both RNG paths (fused and
staged), and full-size properties checked against the CPU oracle."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
from conftest import GOLDEN, bis_case, fill_case

pytestmark = pytest.mark.gpu

with np.load(GOLDEN) as _z:
    N_FILL = len(_z["fill_names"])
    N_BIS = len(_z["bis_names"])


@pytest.fixture(scope="module")
def ctx():
    return _capi.context(0)


_DEFAULTS = {"force_tpb": 0, "no_placement": 0, "no_pdl": 0, "no_step2": 0, "fused_gen": 0,
             "batch_chunk": 0, "no_row_plan": 0, "no_ts": 0, "ts_staged": 0, "no_ts_probe": 0,
             "no_device_loop": 0}


@pytest.fixture
def tuned(ctx):
    """Set rg_set_option knobs on the shared context; restored to the defaults after."""
    def set_(**opts):
        for k, v in opts.items():
            ctx.set_option(k, v)
    yield set_
    set_(**_DEFAULTS)


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def _problem(lower, upper, anchor, eps, j_star):
    tight = rg.tighten(rg.ConstraintSet(lower, upper, anchor), eps)
    lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
    return _capi.Problem(0.01, lower, upper, lo, hi, j_star, 0)


def test_lockstep_tanh_bit_exact(ctx, orc):
    rng = np.random.default_rng(17)
    x = np.concatenate([
        rng.uniform(-1.2, 1.2, 2_000_000), rng.uniform(-7, 7, 1_000_000),
        rng.uniform(-30, 30, 100_000),
        np.ldexp(rng.uniform(0.5, 1.0, 200_000), rng.integers(-64, 6, 200_000)),
        -np.ldexp(rng.uniform(0.5, 1.0, 200_000), rng.integers(-64, 6, 200_000)),
        np.array([0.0, -0.0, np.inf, -np.inf, 22.0, -22.0, 6.5, -6.5, 5e-324, 1.0, -1.0,
                  0.17328679513998632, 0.5198603854199589]),
    ])
    ref = orc.libm_tanh(x)
    y = ctx.tanh(x, lockstep=True)
    mism = np.flatnonzero(_bits(y) != _bits(ref))
    assert mism.size == 0, f"{mism.size} mismatches, first x={x[mism[:5]]}"


def test_small_range_tanh_bit_exact(ctx, orc):
    """The warp-voted small-argument form (|x| < 0.51986, tanh_lockstep_small):
    whole warps of in-range arguments, the k = 0 / k = -1 boundary word, the
    range's last hi word and the 2^-55 floor, each with random low words."""
    rng = np.random.default_rng(23)

    def words(hi, n):
        lo = rng.integers(0, 2**32, n, dtype=np.uint64)
        return ((np.uint64(hi) << np.uint64(32)) | lo).view(np.float64)

    parts = [rng.uniform(-0.5198, 0.5198, 2_000_000),
             rng.uniform(-0.2, 0.2, 500_000),
             np.ldexp(rng.uniform(0.5, 1.0, 200_000), rng.integers(-54, -1, 200_000))]
    for hi in (0x3FC62E41, 0x3FC62E42, 0x3FC62E43, 0x3FE0A2B1, 0x3C800000, 0x3C800001):
        w = words(hi, 128 * 512)
        parts += [w, -w]
    x = np.concatenate(parts)
    ref = orc.libm_tanh(x)
    y = ctx.tanh(x, lockstep=True)
    mism = np.flatnonzero(_bits(y) != _bits(ref))
    assert mism.size == 0, f"{mism.size} mismatches, first x={x[mism[:5]]}"
    # and mixed warps: small arguments next to one out-of-range argument per warp
    x2 = rng.uniform(-0.5, 0.5, 128 * 4096)
    x2[::128] = rng.uniform(0.6, 5.0, 4096)
    y2 = ctx.tanh(x2, lockstep=True)
    assert np.array_equal(_bits(y2), _bits(orc.libm_tanh(x2)))


def test_big_range_tanh_bit_exact(ctx, orc):
    """The warp-voted 1 <= |x| < 6.5 form (tanh_lockstep_big): whole warps in range,
    the range's first and last hi words, every reduction index k = 3..19."""
    rng = np.random.default_rng(29)

    def words(hi, n):
        lo = rng.integers(0, 2**32, n, dtype=np.uint64)
        return ((np.uint64(hi) << np.uint64(32)) | lo).view(np.float64)

    parts = [rng.uniform(1.0, 6.5, 2_000_000), rng.uniform(-6.5, -1.0, 500_000)]
    for hi in (0x3FF00000, 0x3FF00001, 0x40199999, 0x40199FFF):
        w = words(hi, 128 * 512)
        parts += [w, -w]
    # arguments around every k boundary: y = 2|x| = (k - 0.5) ln2
    for k in range(3, 20):
        b = (k - 0.5) * np.log(2.0) / 2.0
        parts.append(b * (1.0 + rng.uniform(-1e-12, 1e-12, 128 * 64)))
    x = np.concatenate(parts)
    x = x[np.abs(x) < 6.5]
    x = x[: x.size // 128 * 128]
    ref = orc.libm_tanh(x)
    y = ctx.tanh(x, lockstep=True)
    mism = np.flatnonzero(_bits(y) != _bits(ref))
    assert mism.size == 0, f"{mism.size} mismatches, first x={x[mism[:5]]}"


@pytest.mark.parametrize("mode", ["fused", "staged"])
@pytest.mark.parametrize("idx", range(N_FILL))
def test_grid_step_both_rng_paths(ctx, golden, idx, mode):
    c = fill_case(golden, idx)
    m = rg.DisturbanceModel(c["ranges"])
    scen = _capi.make_scenarios(c["seed"], 0, c["n_sim"], m.lo, m.span)
    prob = _problem(c["lower"], c["upper"], c["anchor"], c["eps"], c["j_star"])
    res, viol, pbits = ctx.grid_step(prob, c["x0"], c["v_prev"], c["r"], c["m_grid"],
                                     c["prefix"], None, c["n_sim"], scen, True, rng_mode=mode)
    P = np.unpackbits(pbits.view(np.uint8), axis=1, bitorder="little")[:, :c["n_sim"]]
    ss = c["ss_ok"]
    # simulated rows carry their own bits; the reference's P has the same rows
    sim = np.array([i for i in range(c["m_grid"]) if ss[i] and
                    rg.update_setpoint(c["v_prev"], c["r"], i / (c["m_grid"] - 1)) not in
                    [rg.update_setpoint(c["v_prev"], c["r"], q / (c["m_grid"] - 1))
                     for q in range(i) if ss[q]]], dtype=int)
    assert np.array_equal(P[sim].astype(bool), c["P"][sim]), c["name"]
    assert int(res.sims_run) == int(c["stats"][0]) and int(res.early_terms) == int(c["stats"][1])
    kappa = 0.0 if res.row < 0 else res.row / (c["m_grid"] - 1)
    assert kappa == c["result"][0]


@pytest.mark.parametrize("mode", ["fused", "staged"])
@pytest.mark.parametrize("idx", range(N_BIS))
def test_bisect_both_rng_paths(ctx, golden, idx, mode):
    c = bis_case(golden, idx)
    m = rg.DisturbanceModel(c["ranges"])
    scen = _capi.make_scenarios(c["seed"], 0, c["n_sim"], m.lo, m.span)
    prob = _problem(c["lower"], c["upper"], c["anchor"], c["eps"], c["j_star"])
    res, per, paths = ctx.bisect(prob, c["x0"], c["v_prev"], c["r"], c["n_kappa"], None,
                                 c["n_sim"], scen, per_scenario=True, paths=True,
                                 rng_mode=mode)
    pk, po = paths
    ref_k = c["paths"][..., 0]
    used = ~np.isnan(ref_k)
    assert np.array_equal(pk[used], ref_k[used]) and np.array_equal(np.isnan(pk), ~used)
    assert np.array_equal(po[used], c["paths"][..., 1][used].astype(np.uint8))
    assert np.array_equal(np.stack(per, axis=1).astype(np.float64), c["per"]), c["name"]
    assert (res.kappa, float(res.found), res.cells, res.early) == \
        (c["result"][0], c["result"][2], c["result"][3], c["result"][4])


def test_million_scenarios_shard_invariance_and_spot_checks(ctx, orc):
    """C4 shape at reduced horizon: 2^20 scenarios, fused RNG.  Per-row violation
    counts of the whole set equal the sum over four k0-shards (the multi-GPU
    partition), and random cells match the oracle's on-the-fly rollout."""
    n, j_star, M = 1 << 20, 64, 16
    ranges = [(-0.02, 0.02)] * 3
    m = rg.DisturbanceModel(ranges)
    x0 = np.array([np.tanh(0.2), 0.2, np.tanh(0.2) / 2]) + 0.03
    prob = _problem(-0.9, 0.9, 0.0, 0.05, j_star)
    full = _capi.make_scenarios(99, 0, n, m.lo, m.span)
    res, viol, _ = ctx.grid_step(prob, x0, 0.2, 2.4, M, False, None, n, full, False,
                                 rng_mode="fused")
    parts = np.zeros(M, dtype=np.int64)
    for r in range(4):
        sh = _capi.make_scenarios(99, r * n // 4, n // 4, m.lo, m.span)
        _, v, _ = ctx.grid_step(prob, x0, 0.2, 2.4, M, False, None, n // 4, sh, False,
                                rng_mode="fused")
        parts += np.where(v == 0xFFFFFFFF, 0, v)
    assert np.array_equal(np.where(viol == 0xFFFFFFFF, 0, viol).astype(np.int64), parts)
    assert 0 < np.count_nonzero(viol == 0) < M   # the case binds: some rows fail
    # spot-check cells of the failing and passing rows against the oracle
    rng = np.random.default_rng(0)
    ks = rng.choice(n, size=48, replace=False)
    v_rows = np.array([rg.update_setpoint(0.2, 2.4, i / (M - 1)) for i in range(M)])
    rows = np.arange(M, dtype=np.int32)
    for k in ks:
        sc = _capi.make_scenarios(99, int(k), 1, m.lo, m.span)
        S = np.zeros((M, 1), np.uint8)
        st = np.zeros((M, 1), np.int32)
        ctx.fill(prob, x0, v_rows, rows, None, 1, sc, S, st, rng_mode="fused")
        for i in range(0, M, 5):
            assert (int(S[i, 0]), int(st[i, 0])) == orc.cell_sfc_rng(
                0.01, x0, v_rows[i], 99, int(k), ranges, j_star, -0.9, 0.9)


def test_staged_and_fused_agree_at_scale(ctx):
    n, j_star, M = 20_000, 256, 32
    m = rg.DisturbanceModel.scaled(0.02, 3)
    x0 = np.array([np.tanh(-0.4), -0.4, np.tanh(-0.4) / 2])
    prob = _problem(-0.9, 0.9, 0.0, 0.05, j_star)
    sc = _capi.make_scenarios(5, 0, n, m.lo, m.span)
    a = ctx.grid_step(prob, x0, -0.4, -2.5, M, False, None, n, sc, True, rng_mode="fused")
    b = ctx.grid_step(prob, x0, -0.4, -2.5, M, False, None, n, sc, True, rng_mode="staged")
    assert a[0].row == b[0].row and a[0].early_terms == b[0].early_terms
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


@pytest.mark.parametrize("idx", range(N_FILL))
def test_fill_cells_all_rows(ctx, golden, idx):
    c = fill_case(golden, idx)
    grid = rg.grid_kappas(c["m_grid"])
    v_rows = np.array([rg.update_setpoint(c["v_prev"], c["r"], float(k)) for k in grid])
    S = np.full((c["m_grid"], c["n_sim"]), 7, np.uint8)
    steps = np.full((c["m_grid"], c["n_sim"]), -1, np.int32)
    m = rg.DisturbanceModel(c["ranges"])
    scen = _capi.make_scenarios(c["seed"], 0, c["n_sim"], m.lo, m.span)
    ctx.fill(_problem(c["lower"], c["upper"], c["anchor"], c["eps"], c["j_star"]), c["x0"],
             v_rows, np.arange(c["m_grid"], dtype=np.int32), None, c["n_sim"], scen, S, steps)
    assert np.array_equal(S, c["S_all"]) and np.array_equal(steps, c["steps_all"]), c["name"]


@pytest.mark.parametrize("abandon", [False, True])
@pytest.mark.parametrize("chunk", [None, 5, 1])
def test_batch_staged_chunks_equal_fused(ctx, tuned, chunk, abandon):
    """Staged episode blocks (k_gen_soa_batch), in one or several chunks of
    episodes, against the fused in-rollout RNG: same rows, kappas, setpoints,
    early counts and per-row violation counts."""
    if chunk is not None:
        tuned(batch_chunk=chunk)
    rng = np.random.default_rng(11)
    E, n, M = 13, 150, 8
    vp = rng.uniform(-1, 1, E)
    r = rng.uniform(-2.5, 2.5, E)
    X = np.stack([[np.tanh(v), v, np.tanh(v) / 2] for v in vp]) + rng.uniform(-0.05, 0.05, (E, 3))
    seeds = [int(x) for x in rng.integers(0, 2**63, E)]
    m = rg.DisturbanceModel.scaled(0.02, 3)
    prob = _problem(-0.9, 0.9, 0.0, 0.05, 64)
    ref = ctx.grid_step_batch(prob, X, vp, r, seeds, 7, n, m.lo, m.span, M, abandon=abandon,
                              want_viol=not abandon, fused=True)
    got = ctx.grid_step_batch(prob, X, vp, r, seeds, 7, n, m.lo, m.span, M, abandon=abandon,
                              want_viol=not abandon, staged=True)
    for a, b in zip(ref, got):
        assert np.array_equal(a, b)


def test_grid_fetch_after_sync_and_async_steps(ctx):
    """rg_grid_fetch returns the LAST step's result: after a synchronous (zero-copy)
    step it re-reads that step; after an RG_ASYNC step on different inputs it returns
    the async step's result, not the pinned block of the synchronous one before it."""
    import ctypes

    m = rg.DisturbanceModel.scaled(0.02, 3)
    prob = _problem(-0.9, 0.9, 0.0, 0.05, 128)
    x0 = np.array([0.1, 0.3, 0.05])
    sc_a = _capi.make_scenarios(77, 0, 3000, m.lo, m.span)
    sc_b = _capi.make_scenarios(78, 0, 3000, m.lo, m.span)
    lib = ctx.lib
    # reference results of both inputs, each from its own synchronous step
    res_b, viol_b, _ = ctx.grid_step(prob, x0, 0.3, 1.9, 32, False, None, 3000, sc_b, False)
    res_a, viol_a, _ = ctx.grid_step(prob, x0, 0.3, 2.4, 32, False, None, 3000, sc_a, False)
    assert not np.array_equal(viol_a, viol_b), "the two inputs must give different counts"

    def fetch():
        got = _capi.GridResult()
        v2 = np.empty(32, np.uint32)
        _capi.check(lib.rg_grid_fetch(ctx.handle, v2.ctypes.data, 32, ctypes.byref(got)))
        return got, v2

    got, v2 = fetch()  # after the synchronous step on inputs a
    assert (got.row, got.sims_run, got.early_terms, got.overflows) == \
        (res_a.row, res_a.sims_run, res_a.early_terms, res_a.overflows)
    assert np.array_equal(v2, viol_a)
    out = _capi.GridResult()
    _capi.check(lib.rg_grid_step(ctx.handle, ctypes.byref(prob), x0.ctypes.data, 0.3, 1.9, 32, 0,
                                 None, 3000, 0, ctypes.byref(sc_b), None, None,
                                 ctypes.byref(out), _capi.RG_ASYNC))
    got, v2 = fetch()  # after the asynchronous step on inputs b
    assert (got.row, got.sims_run, got.early_terms, got.overflows) == \
        (res_b.row, res_b.sims_run, res_b.early_terms, res_b.overflows)
    assert np.array_equal(v2, viol_b)


@pytest.mark.parametrize("opts", [{"no_placement": 1}, {"force_tpb": 32}, {"force_tpb": 128},
                                  {"no_step2": 1}, {"no_pdl": 1}, {"fused_gen": 1}])
@pytest.mark.parametrize("shape", [(1000, 32), (300, 32), (4000, 32), (97, 5)])
def test_single_wave_placement_changes_no_bit(ctx, tuned, opts, shape):
    """The single-wave placement (blocks of 4L warps pinned one per SM, with the
    two-step rollout over the staged block) against the other block shapes and the
    one-step rollout (the multi-wave forms), on transient-binding inputs: same P
    bits, per-row counts, result row and counters; and the same for the bisections."""
    n, M = shape
    rng = np.random.default_rng(n + M)
    vp = 0.4
    x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.05, 0.05, 3)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    scen = _capi.make_scenarios(4242 + n, 0, n, m.lo, m.span)
    prob = _problem(-0.9, 0.9, 0.0, 0.05, 256)

    def run():
        res, viol, pbits = ctx.grid_step(prob, x0, vp, 2.4, M, False, None, n, scen, True)
        b, _, _ = ctx.bisect(prob, x0, vp, 2.4, 8, None, n, scen)
        j = ctx.bisect_joint(prob, x0, vp, 2.4, 8, None, n, scen)
        return (res.row, res.sims_run, res.early_terms, res.overflows, viol.copy(),
                pbits.copy(), b.kappa, b.found, b.cells, b.early, j.kappa, j.found, j.cells)

    ref = run()
    tuned(**opts)
    got = run()
    assert ref[1] > 0 and 0 < int(np.count_nonzero(ref[4])) , "inputs must bind some rows"
    for a, b in zip(ref, got):
        assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("j_star", [1, 2, 3, 31, 32, 33, 64, 257])
@pytest.mark.parametrize("shape", [(1000, 32), (300, 8)])
def test_two_step_rollout_edges(ctx, tuned, shape, j_star):
    """The single-wave two-step rollout (rollout2) at odd and short horizons, with
    and without abandonment (the polled form), against the one-step rollout."""
    n, M = shape
    m = rg.DisturbanceModel.scaled(0.02, 3)
    prob = _problem(-0.9, 0.9, 0.0, 0.05, j_star)
    rng = np.random.default_rng(j_star * 7 + n)
    cases = []
    for trial in range(3):
        vp = float(rng.uniform(-1, 1))
        r = float(rng.uniform(-2.5, 2.5))
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.05, 0.05, 3)
        cases.append((vp, r, x0, _capi.make_scenarios(500 + trial, 0, n, m.lo, m.span)))

    def run():
        out = []
        for vp, r, x0, sc in cases:
            a = ctx.grid_step(prob, x0, vp, r, M, False, None, n, sc, True)
            b = ctx.grid_step(prob, x0, vp, r, M, False, None, n, sc, False, abandon=True)
            out.append((a[0].row, a[0].early_terms, a[0].overflows, a[0].sims_run, a[1].copy(),
                        a[2].copy(), b[0].row, b[1] == 0))
        return out

    got = run()
    tuned(no_step2=1)
    ref = run()
    for g, f in zip(got, ref):
        for x, y in zip(g, f):
            assert np.array_equal(np.asarray(x), np.asarray(y))
        assert g[6] == g[0]  # abandonment changes no verdict


def test_concurrent_calls_on_one_context_are_serialised():
    """The reference service runs /govern/step in a thread pool: concurrent governor
    calls on one device (one shared context) must each get their own result --
    the same as the calls made one after another."""
    from concurrent.futures import ThreadPoolExecutor

    plant = rg.make_plant("surrogate-fc")
    box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
    model = rg.DisturbanceModel.scaled(0.02, 3)
    cfg = rg.GovernorConfig(j_star=128, n_sim=2000, m_grid=32, n_kappa=8)
    rng = np.random.default_rng(5)
    jobs = []
    for q in range(16):
        vp = float(rng.uniform(-1, 1))
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.05, 0.05, 3)
        jobs.append((x0, vp, float(rng.uniform(-2.5, 2.5)), 900 + q))

    def call(job):
        x0, vp, r, seed = job
        scen = rg.sample_scenarios(model, cfg.n_sim, cfg.j_star + 1, seed=seed)
        a = rg.robust_rg_parallel(plant, x0, rg.GovernorState(vp), r, box, scen, cfg)
        b = rg.robust_rg_sequential(plant, x0, rg.GovernorState(vp), r, box, scen, cfg)
        return a.kappa_opt, a.v_applied, a.feasible, a.matrix.copy(), b.kappa_opt, \
            b.diagnostics["sims_run"]

    serial = [call(j) for j in jobs]
    for _ in range(3):
        with ThreadPoolExecutor(max_workers=8) as ex:
            conc = list(ex.map(call, jobs))
        for s_, c_ in zip(serial, conc):
            assert s_[:3] == c_[:3] and np.array_equal(s_[3], c_[3]) and s_[4:] == c_[4:]


@pytest.mark.parametrize("rng_mode", ["auto", "fused", "staged"])
@pytest.mark.parametrize("prefix", [False, True])
def test_batch_pairs_equal_single_steps(ctx, tuned, rng_mode, prefix):
    """The compacted batched step (host gate + dedup, one launch over the live (episode,
    row) pairs) against one rg_grid_step per episode on the same stream: every episode's
    row, kappa, v, early count and per-row counts -- with episodes whose rows are all
    duplicates (v_prev == r), all gated out (nothing runs), partly violating, and staged
    chunks of a few episodes."""
    rng = np.random.default_rng(77)
    E, n, M = 41, 333, 32
    vp = rng.uniform(-1.2, 1.2, E)
    r = rng.uniform(-3.0, 3.0, E)
    r[:5] = vp[:5]                      # all rows the same setpoint
    vp[5:8], r[5:8] = 2.9, 2.95         # every row gated out
    X = np.stack([[np.tanh(v), v, np.tanh(v) / 2] for v in vp]) + rng.uniform(-0.06, 0.06,
                                                                               (E, 3))
    seeds = [int(x) for x in rng.integers(0, 2**63, E)]
    m = rg.DisturbanceModel.scaled(0.02, 3)
    prob = _problem(-0.9, 0.9, 0.0, 0.05, 96)
    if rng_mode == "staged":
        tuned(batch_chunk=4)
    kw = {"fused": rng_mode == "fused", "staged": rng_mode == "staged"}
    row, kap, v, early, viol = ctx.grid_step_batch(prob, X, vp, r, seeds, 5, n, m.lo, m.span, M,
                                                   prefix_mode=prefix, abandon=False,
                                                   want_viol=True, **kw)
    for e in range(E):
        sc = _capi.make_scenarios(seeds[e], 5, n, m.lo, m.span)
        res, vi, _ = ctx.grid_step(prob, X[e], vp[e], r[e], M, prefix, None, n, sc, False)
        assert row[e] == res.row and early[e] == res.early_terms, e
        assert np.array_equal(viol[e], vi), e
        k = 0.0 if res.row < 0 else res.row / (M - 1)
        assert kap[e] == k and v[e] == (vp[e] if res.row < 0 else rg.update_setpoint(vp[e], r[e], k))
    ab = ctx.grid_step_batch(prob, X, vp, r, seeds, 5, n, m.lo, m.span, M, prefix_mode=prefix,
                             abandon=True, **kw)
    assert np.array_equal(ab[0], row) and np.array_equal(ab[1], kap) and np.array_equal(ab[2], v)


@pytest.mark.parametrize("n", [1, 31, 97, 1000, 4099])
def test_dense_host_tensor_staging_equals_generated(ctx, n):
    """A caller's dense host tensor goes through pinned staging in chunks of scenarios
    (parallel host copies, async DMA, per-chunk transposes): every size, including chunk
    tails and padding, gives the generated stream's bits, twice in a row (staging reuse)."""
    m = rg.DisturbanceModel.scaled(0.02, 3)
    prob = _problem(-0.9, 0.9, 0.0, 0.05, 200)
    x0 = np.array([0.12, 0.3, 0.07])
    sc = _capi.make_scenarios(4040 + n, 0, n, m.lo, m.span)
    dense = rg.sample_scenarios(m, n, 201, seed=4040 + n).data
    ref = ctx.grid_step(prob, x0, 0.3, 2.2, 32, False, None, n, sc, True)
    for _ in range(2):
        got = ctx.grid_step(prob, x0, 0.3, 2.2, 32, False, dense, n, None, True)
        assert got[0].row == ref[0].row and got[0].early_terms == ref[0].early_terms
        assert np.array_equal(got[1], ref[1]) and np.array_equal(got[2], ref[2])
    b_ref = ctx.bisect(prob, x0, 0.3, 2.2, 8, None, n, sc)[0]
    b_got = ctx.bisect(prob, x0, 0.3, 2.2, 8, dense, n, None)[0]
    assert (b_got.kappa, b_got.found, b_got.cells, b_got.early) == \
        (b_ref.kappa, b_ref.found, b_ref.cells, b_ref.early)


@pytest.mark.parametrize("n", [1, 300, 1000, 10_000])
def test_host_row_plan_equals_device_rows(ctx, tuned, n):
    """Grid steps without P launch only the host-planned simulated rows (closed-loop steps
    have about one); against the device-derived rows: same row, per-row counts (gated -1,
    duplicates their source's), early / overflow counts and row statistics -- in random
    transient cases with gated and duplicate rows, with and without abandonment."""
    rng = np.random.default_rng(n)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    cases = []
    for trial in range(16):
        vp = float(rng.uniform(-1.2, 1.2))
        r = [float(rng.uniform(-3, 3)), vp, vp + 1e-3, 2.9][trial % 4]
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.06, 0.06, 3)
        M = int(rng.choice([2, 8, 32, 64]))
        cases.append((vp, r, x0, M, bool(trial % 3 == 2),
                      _capi.make_scenarios(300 + trial, 0, n, m.lo, m.span)))
    prob = _problem(-0.9, 0.9, 0.0, 0.05, 128)

    def run():
        out = []
        for vp, r, x0, M, prefix, sc in cases:
            for abandon in (False, True):
                res, viol, _ = ctx.grid_step(prob, x0, vp, r, M, prefix, None, n, sc, False,
                                             abandon=abandon)
                out.append((res.row, res.sims_run, res.ss_pruned_rows, res.dedup_rows,
                            res.n_active, (viol == 0).tolist(),
                            None if abandon else (viol.tolist(), res.early_terms,
                                                  res.overflows)))
        return out

    planned = run()
    tuned(no_row_plan=1)
    device = run()
    assert planned == device


@pytest.mark.parametrize("j_star", [1, 5, 8, 9, 17, 256])
@pytest.mark.parametrize("n", [1, 33, 1000, 10_000, 13_000])
def test_time_split_step_equals_k_grid(ctx, tuned, n, j_star):
    """Host-planned steps whose cells fit one wave run the time-split kernel (rg_ts.cu: the
    x2 chain, the tanh and the x1/x3 chain on separate warps; generated scenarios by the
    producer's fused RNG or through the staged block); against k_grid (no_ts):
    the same row, per-row violation counts, early-termination and overflow counts -- in
    transient cases (violations at every step count, out-of-bounds starts, overflowing
    states), from generated and from dense host scenarios, chunk-ragged horizons."""
    rng = np.random.default_rng(7 * n + j_star)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    prob = _problem(-0.9, 0.9, 0.0, 0.05, j_star)
    cases = []
    for trial in range(6):
        vp = float(rng.uniform(-1.2, 1.2))
        # r == vp: every candidate is vp, one simulated row (the closed loop's steady state)
        r = [float(rng.uniform(-3, 3)), vp + 1e-3, vp][trial % 3]
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.08, 0.08, 3)
        if trial == 4:
            x0[0] = 0.95  # out of bounds at the start: steps 0
        if trial == 5:
            x0[2] = 1.5e6  # beyond STATE_LIMIT: the first step overflows
        cases.append((vp, r, x0, [8, 32][trial % 2], trial % 4 == 3,
                      _capi.make_scenarios(900 + trial, 0, n, m.lo, m.span)))
    dense = rg.sample_scenarios(m, n, j_star + 1, seed=77).data

    kernels = []

    def run():
        out = []
        for vp, r, x0, M, prefix, sc in cases:
            for dist, scen in ((None, sc), (dense, None)):
                res, viol, _ = ctx.grid_step(prob, x0, vp, r, M, prefix, dist, n, scen, False)
                out.append((res.row, res.sims_run, res.n_active, viol.tolist(),
                            res.early_terms, res.overflows))
                kernels.append(ctx.get_option("last_grid_kernel"))
        return out

    ts = run()  # generated scenarios: the producer's fused RNG; dense: the staged block
    assert 1 in kernels  # the time-split kernel ran (one wave holds <= 3 units per SM)
    tuned(ts_staged=1)
    assert run() == ts  # generated scenarios through the staged block
    tuned(no_ts=1)
    kernels.clear()
    ref = run()
    assert set(kernels) == {0}
    assert ts == ref
    # the cases exercise the verdict paths: some violations, some overflow
    assert any(o[4] > 0 for o in ref) and any(o[5] > 0 for o in ref)


def test_grid_step_kernel_count(ctx, tuned):
    """rg_get_option("grid_step_kernels") counts what a grid step launched: a closed-loop
    step (one live row; with or without P) is one time-split kernel generating its own
    scenarios; a step with every row live stages its block first (generator + k_grid); with
    ts_staged the time-split step reads a staged block too."""
    m = rg.DisturbanceModel.scaled(0.001, 3)
    prob = _problem(-0.9, 0.9, 0.0, 0.05, 256)
    vp = 0.4
    x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2])
    sc = _capi.make_scenarios(5, 0, 10_000, m.lo, m.span)

    def count(r, want_pbits=False):
        k0 = ctx.get_option("grid_step_kernels")
        ctx.grid_step(prob, x0, vp, r, 32, False, None, 10_000, sc, want_pbits)
        return ctx.get_option("grid_step_kernels") - k0, ctx.get_option("last_grid_kernel")

    assert count(vp) == (1, 1)             # one live row: k_grid_ts, fused RNG
    assert count(vp, want_pbits=True) == (1, 1)  # with P too (the other rows' words zeroed)
    assert count(vp + 0.3) == (2, 0)       # 32 distinct live rows: staged block + k_grid
    tuned(ts_staged=1)
    assert count(vp) == (2, 1)


def test_options_round_trip(ctx, tuned):
    """rg_get_option reads back every rg_set_option knob; unknown names are ConfigError."""
    from paper_2510_08288_b200.errors import ConfigError

    for name, value in (("force_tpb", 64), ("no_placement", 1), ("no_pdl", 1), ("no_step2", 1),
                        ("fused_gen", 1), ("no_row_plan", 1), ("no_ts", 1), ("ts_staged", 1),
                        ("no_ts_probe", 1), ("no_device_loop", 1),
                        ("batch_chunk", 7), ("xchg_timeout_ms", 1234)):
        before = ctx.get_option(name)
        ctx.set_option(name, value)
        assert ctx.get_option(name) == value
        ctx.set_option(name, before)
    with pytest.raises(ConfigError):
        ctx.get_option("no_such_knob")
    with pytest.raises(ConfigError):
        ctx.set_option("last_grid_kernel", 1)  # read-only


def test_time_split_random_stress(ctx, tuned):
    """150 random one- and few-row steps (scenario counts 1..13,000, horizons 1..300,
    random starts, setpoints, disturbance scales and grid sizes): the time-split kernel
    (fused RNG and staged) gives k_grid's row, per-row violation counts, early and overflow
    counts on every one."""
    rng = np.random.default_rng(20261019)
    cases = []
    for trial in range(150):
        n = int(rng.choice([1, 7, 31, 32, 33, 500, 1000, 4097, 10_000, 13_000]))
        j = int(rng.choice([1, 2, 7, 8, 9, 15, 16, 17, 64, 255, 256, 300]))
        M = int(rng.choice([2, 5, 16, 32, 64]))
        vp = float(rng.uniform(-1.3, 1.3))
        r = vp if trial % 2 else vp + float(rng.choice([1e-9, 1e-3, 0.3])) * rng.choice([-1, 1])
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.1, 0.1, 3)
        amp = float(rng.choice([0.001, 0.02, 0.08]))
        m = rg.DisturbanceModel.scaled(amp, 3)
        cases.append((_problem(-0.9, 0.9, 0.0, 0.05, j), n, M, vp, r, x0,
                      _capi.make_scenarios(1000 + trial, int(rng.integers(0, 1 << 20)), n, m.lo,
                                           m.span), bool(trial % 5 == 0)))

    def run():
        out, ks = [], []
        for prob, n, M, vp, r, x0, sc, prefix in cases:
            res, viol, _ = ctx.grid_step(prob, x0, vp, r, M, prefix, None, n, sc, False)
            out.append((res.row, res.n_active, res.sims_run, viol.tolist(), res.early_terms,
                        res.overflows))
            ks.append(ctx.get_option("last_grid_kernel"))
        return out, ks

    ts, ks = run()
    assert sum(ks) > 50  # most cases fit the time-split form
    tuned(ts_staged=1)
    staged, _ = run()
    tuned(ts_staged=0, no_ts=1)
    ref, ks_ref = run()
    assert set(ks_ref) == {0}
    assert ts == ref and staged == ref


@pytest.mark.parametrize("n", [33, 1000, 10_000])
def test_row_plan_with_p_equals_device_rows(ctx, tuned, n):
    """Steps that return P also launch only the host-planned rows (time-split or k_grid):
    the gated-out and duplicate rows' words come back zero, so P, the per-row counts and
    the row equal the device-derived rows' -- through robust_rg_parallel's expansion too."""
    rng = np.random.default_rng(n + 3)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    prob = _problem(-0.9, 0.9, 0.0, 0.05, 96)
    cases = []
    for trial in range(8):
        vp = float(rng.uniform(-1.2, 1.2))
        r = [vp, vp + 1e-3, float(rng.uniform(-3, 3)), 2.9][trial % 4]
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.06, 0.06, 3)
        cases.append((vp, r, x0, int(rng.choice([8, 32])), trial % 3 == 1,
                      _capi.make_scenarios(70 + trial, 0, n, m.lo, m.span)))

    def run():
        out = []
        for vp, r, x0, M, prefix, sc in cases:
            res, viol, pb = ctx.grid_step(prob, x0, vp, r, M, prefix, None, n, sc, True)
            out.append((res.row, res.n_active, res.ss_pruned_rows, res.dedup_rows,
                        viol.tolist(), pb.copy()))
        return out

    planned = run()
    tuned(no_row_plan=1)
    device = run()
    for a, b in zip(planned, device):
        assert a[:5] == b[:5]
        assert np.array_equal(a[5], b[5])


@pytest.mark.parametrize("n", [1, 45, 1000, 10_000])
def test_bisect_time_split_probe_equals_inline_probe(ctx, tuned, n):
    """Alg. 2's kappa = 1 probe run ahead by the time-split kernel (its verdict and early bits
    handed to k_bisect) against the probe rolled out inside k_bisect: the same kappa, found,
    cells and early counts, per-scenario results and search paths -- steady states (the
    probe alone), transients (probe failures, then bisection), out-of-bounds starts,
    generated and dense scenarios."""
    rng = np.random.default_rng(11 * n + 1)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    prob = _problem(-0.9, 0.9, 0.0, 0.05, 128)
    dense = rg.sample_scenarios(m, n, 129, seed=5).data
    cases = []
    for trial in range(8):
        vp = float(rng.uniform(-1.1, 1.1))
        r = [vp, float(rng.uniform(-1.2, 1.2)), 2.4, vp + 0.05][trial % 4]
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.08, 0.08, 3)
        if trial == 6:
            x0[0] = 0.93  # out of bounds: every rollout fails at step 0
        cases.append((vp, r, x0, _capi.make_scenarios(40 + trial, 3, n, m.lo, m.span)))

    def run():
        out = []
        for vp, r, x0, sc in cases:
            # generated, dense, and no scenarios (bisection_rg's nominal prediction)
            for dist, scen in ((None, sc), (dense, None), (None, None)):
                b, per, path = ctx.bisect(prob, x0, vp, r, 8, dist, n, scen, per_scenario=True,
                                          paths=True)
                out.append(((b.kappa, b.found, b.cells, b.early),
                            [np.asarray(a).copy() for a in per],
                            [np.asarray(a).copy() for a in path]))
        return out

    probe = run()
    tuned(no_ts_probe=1)
    inline = run()
    for a, b in zip(probe, inline):
        assert a[0] == b[0]
        for x, y in zip(a[1] + a[2], b[1] + b[2]):
            assert np.array_equal(x, y, equal_nan=True)


@pytest.mark.parametrize("n", [1, 500, 1000, 10_000])
def test_joint_time_split_probe_equals_inline_probe(ctx, tuned, n):
    """The persistent joint search's kappa = 1 probe rolled out first by the time-split
    kernel against the probe inside the search: the same kappa, found and rollout count, in
    steady states (the probe alone), gated-in transients and out-of-bounds starts."""
    rng = np.random.default_rng(5 * n + 2)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    prob = _problem(-0.9, 0.9, 0.0, 0.05, 128)
    cases = []
    for trial in range(10):
        vp = float(rng.uniform(-1.1, 1.1))
        r = [vp, float(rng.uniform(-1.2, 1.2)), vp + 0.05, 2.4][trial % 4]
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.08, 0.08, 3)
        if trial == 5:
            x0[0] = 0.93
        cases.append((vp, r, x0, _capi.make_scenarios(60 + trial, 0, n, m.lo, m.span)))

    def run():
        out = []
        for vp, r, x0, sc in cases:
            for scen in (sc, None):  # generated, and the nominal prediction
                j = ctx.bisect_joint(prob, x0, vp, r, 8, None, n, scen)
                out.append((j.kappa, j.found, j.cells))
        return out

    probe = run()
    tuned(no_ts_probe=1)
    inline = run()
    assert probe == inline
