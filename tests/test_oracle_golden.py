"""Pin the CPU oracle (oracle/) to the real reference's outputs (tests/golden/).

CPU-only.  Every fixture was produced by the reference package itself
(tests/golden/make_golden.py); the oracle must reproduce each bit exactly
before anything else is compared against it.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, bis_case, fill_case, lin_case

with np.load(GOLDEN) as _z:
    N_FILL = len(_z["fill_names"])
    N_BIS = len(_z["bis_names"])

MASK = (1 << 64) - 1


def test_splitmix_published_sequence(orc, golden):
    # tests/test_disturbance.py:28-34 of the reference
    seq = [orc.splitmix64((n * 0x9E3779B97F4A7C15) & MASK) for n in range(3)]
    assert seq == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert seq == [int(v) for v in golden["sm_seed0"]]
    for z, out in zip(golden["sm_in"], golden["sm_out"]):
        assert orc.splitmix64(int(z)) == int(out)


def test_counter_uniform_and_derive_seed(orc, golden):
    for row, out in zip(golden["cu_coords"], golden["cu_out"]):
        assert orc.counter_uniform(*(int(c) for c in row)) == out
    labels = [str(s) for s in golden["derive_labels"]]
    got = [orc.derive_seed(2024, lb) for lb in labels] + [orc.derive_seed(MASK, "plant")]
    assert got == [int(v) for v in golden["derive_out"]]


def test_sample_scenarios_bit_exact(orc, golden):
    ranges = ((-0.003, 0.001), (0.0, 0.002), (-1e-4, 1e-4))
    assert np.array_equal(orc.sample(2**63 + 5, 5, 9, ranges), golden["scen_small"])
    u = orc.uniform_grid(2**64 - 3, 4, 6, 3, k0=1_000_000)
    assert np.array_equal(u, golden["scen_small_k0"])
    big = orc.sample(7, 1000, 257, [(-0.001, 0.001)] * 3)
    assert hashlib.sha256(big.tobytes()).digest() == golden["scen_big_sha"].tobytes()
    assert np.array_equal(big[[0, 1, 511, 999]], golden["scen_big_rows"])
    wrap = orc.sample(((MASK - 1) + 5) & MASK, 3, 5, [(-0.001, 0.001)] * 3)
    assert np.array_equal(wrap, golden["scen_wrap"])


def test_sample_chunk_and_prefix_invariance(orc):
    whole = orc.uniform_grid(5, 50, 7, 3)
    parts = np.concatenate([orc.uniform_grid(5, 20, 7, 3), orc.uniform_grid(5, 30, 7, 3,
                                                                           k0=20)])
    assert np.array_equal(whole, parts)


def test_libm_tanh_matches_reference_host(orc, golden):
    # The oracle binds the same glibc tanh numba calls (kernels.py:56).
    y = orc.libm_tanh(golden["tanh_x"])
    assert np.array_equal(y.view(np.uint64), golden["tanh_libm"].view(np.uint64))


@pytest.mark.parametrize("idx", range(N_FILL))
def test_fill_cells_match_reference(orc, golden, idx):
    c = fill_case(golden, idx)
    dist = orc.sample(c["seed"], c["n_sim"], c["j_star"] + 1, c["ranges"])
    grid = orc.grid_kappas(c["m_grid"])
    v_rows = np.array([orc.update_setpoint(c["v_prev"], c["r"], float(k)) for k in grid])
    S = np.zeros((c["m_grid"], c["n_sim"]), np.uint8)
    steps = np.zeros((c["m_grid"], c["n_sim"]), np.int32)
    for workers in (1, 3):
        orc.run_cells(0.01, c["x0"], v_rows, np.arange(c["m_grid"]), dist, c["j_star"],
                      c["lower"], c["upper"], S, steps, workers=workers)
        assert np.array_equal(S, c["S_all"]), c["name"]
        assert np.array_equal(steps, c["steps_all"]), c["name"]


@pytest.mark.parametrize("idx", range(N_FILL))
def test_fill_feasibility_matches_reference(orc, golden, idx):
    c = fill_case(golden, idx)
    dist = orc.sample(c["seed"], c["n_sim"], c["j_star"] + 1, c["ranges"])
    tlo, thi = orc.tighten(c["lower"], c["upper"], c["anchor"], c["eps"])
    P, S, steps, stats = orc.fill_feasibility(
        0.01, c["x0"], c["v_prev"], c["r"], orc.grid_kappas(c["m_grid"]), dist, c["lower"],
        c["upper"], tlo, thi, c["j_star"])
    assert np.array_equal(P, c["P"]), c["name"]
    got = [stats[k] for k in ("sims_run", "early_terms", "overflows", "ss_pruned_rows",
                              "dedup_rows")]
    assert got == [int(v) for v in c["stats"]], c["name"]
    kappa, v, feas, row, _, _ = orc.grid_step(
        0.01, c["x0"], c["v_prev"], c["r"], c["m_grid"], dist, c["lower"], c["upper"], tlo,
        thi, c["j_star"], prefix_mode=c["prefix"])
    assert (kappa, v, float(feas)) == tuple(float(x) for x in c["result"]), c["name"]


def test_fill_cases_exercise_every_status(golden):
    seen = set()
    for i in range(N_FILL):
        seen |= set(np.unique(fill_case(golden, i)["S_all"]).tolist())
    assert seen == {0, 1, 2}


@pytest.mark.parametrize("idx", range(N_BIS))
def test_bisection_matches_reference(orc, golden, idx):
    c = bis_case(golden, idx)
    dist = orc.sample(c["seed"], c["n_sim"], c["j_star"] + 1, c["ranges"])
    tlo, thi = orc.tighten(c["lower"], c["upper"], c["anchor"], c["eps"])
    kappa, v, feas, cells, early, per = orc.robust_sequential(
        0.01, c["x0"], c["v_prev"], c["r"], c["lower"], c["upper"], tlo, thi, dist,
        c["j_star"], c["n_kappa"])
    assert (kappa, v, float(feas), cells, early) == tuple(float(x) for x in c["result"])
    for k, (kk, fk, ck, ek, path) in enumerate(per):
        assert (kk, float(fk), ck, ek) == tuple(c["per"][k]), (c["name"], k)
        ref_path = [(a, bool(b)) for a, b in c["paths"][k] if not np.isnan(a)]
        assert [(a, bool(b)) for a, b in path] == ref_path, (c["name"], k)


def test_nominal_bisection_anchor(orc, golden):
    # r=2.5 from rest gives bisection kappa 0.5078125
    tlo, thi = orc.tighten(-0.9, 0.9, 0.0, 0.05)
    kappa, found, cells, early, _ = orc.bisect_kappa(
        0.01, np.zeros(3), 0.0, 2.5, -0.9, 0.9, tlo, thi, np.zeros((257, 3)), 256, 8)
    assert kappa == 0.5078125
    assert (kappa, 0.0 + 2.5 * kappa, float(found), cells, early) == \
        tuple(float(x) for x in golden["nominal_anchor"])


def test_closed_loop_c1_bisection_trace(orc, golden):
    prof = golden["desk_profile"]
    rows, aborted = orc.closed_loop(0.01, -0.9, 0.9, 0.0, 0.05, [(-0.001, 0.001)] * 3, prof,
                                    2000, 2024, "bisection")
    assert not aborted
    ref = golden["c1_trace"]
    got = np.array([[r[4], r[2], float(r[5]), r[3]] for r in rows])
    assert np.array_equal(got, ref[:, :4])


def test_closed_loop_desk_grid_trace(orc, golden):
    prof = golden["desk_profile"]
    rows, aborted = orc.closed_loop(0.01, -0.9, 0.9, 0.0, 0.05, [(-0.001, 0.001)] * 3, prof,
                                    2000, 2024, "grid", n_sim=64, workers=4)
    assert not aborted
    got = np.array([[r[2], r[3], r[4], float(r[5])] for r in rows])
    assert np.array_equal(got, golden["desk_grid_trace"])


def test_closed_loop_c3_10k_first_steps(orc, golden):
    """The oracle reproduces the first steps of the reference's 10k-scenario C3 trace
    (tests/golden/make_c3_golden.py); the device runs all of it (test_gpu_parity)."""
    with np.load(GOLDEN.with_name("c3_10k_trace.npz")) as z:
        want, n_sim, seed = z["trace"], int(z["n_sim"]), int(z["seed"])
    steps = 6
    sched = golden["desk_profile"][:steps]
    rows, aborted = orc.closed_loop(0.01, -0.9, 0.9, 0.0, 0.05, [(-0.001, 0.001)] * 3, sched,
                                    steps, seed, "grid", n_sim=n_sim, workers=orc.cpu_count())
    assert not aborted
    got = np.array([[r[2], r[3], r[4], float(r[5])] for r in rows])
    assert np.array_equal(got, want[:steps])


with np.load(GOLDEN) as _z:
    N_LIN = len(_z["lin_names"])


@pytest.mark.parametrize("idx", range(N_LIN))
def test_linear_cells_and_governors_match_reference(orc, golden, idx):
    c = lin_case(golden, idx)
    n = c["A"].shape[0]
    dist = orc.sample(c["seed"], c["n_sim"], c["j_star"] + 1, [(-c["mag"], c["mag"])] * n)
    grid = orc.grid_kappas(c["m_grid"])
    for i, kappa in enumerate(grid):
        v = orc.update_setpoint(c["v_prev"], c["r"], float(kappa))
        for k in range(c["n_sim"]):
            assert orc.cell_lin(c["A"], c["B"], c["C"], c["D"], c["x0"], v, dist[k],
                                c["j_star"], c["lower"], c["upper"]) == \
                (int(c["S_all"][i, k]), int(c["steps_all"][i, k])), (c["name"], i, k)
    tlo, thi = orc.tighten(c["lower"], c["upper"], c["anchor"], c["eps"])
    P, _, _ = orc.fill_feasibility_lin(c["A"], c["B"], c["C"], c["D"], c["gain"], c["x0"],
                                       c["v_prev"], c["r"], grid, dist, c["lower"], c["upper"],
                                       tlo, thi, c["j_star"])
    assert np.array_equal(P, c["P"]), c["name"]
    kap = [orc.bisect_kappa_lin(c["A"], c["B"], c["C"], c["D"], c["gain"], c["x0"],
                                c["v_prev"], c["r"], c["lower"], c["upper"], tlo, thi, dist[k],
                                c["j_star"], 8) for k in range(c["n_sim"])]
    assert min(min(k[0] for k in kap), 1.0) == c["results"][3]
    assert sum(k[2] for k in kap) == c["results"][6] and sum(k[3] for k in kap) == \
        c["results"][7]


def test_linear_known_answer(golden):
    assert abs(float(golden["lin_kappa_star_081"][0]) - 0.81) < 1e-5


@pytest.mark.parametrize("idx", range(N_BIS))
def test_joint_bisection_equals_alg2_on_reference_cases(orc, golden, idx):
    # with down-set feasible sets the joint search
    # (one kappa for all scenarios per iteration) lands on Alg. 2's minimum
    c = bis_case(golden, idx)
    dist = orc.sample(c["seed"], c["n_sim"], c["j_star"] + 1, c["ranges"])
    tlo, thi = orc.tighten(c["lower"], c["upper"], c["anchor"], c["eps"])
    kappa, found, path = orc.joint_bisect(0.01, c["x0"], c["v_prev"], c["r"], c["lower"],
                                          c["upper"], tlo, thi, dist, c["j_star"], c["n_kappa"])
    assert (kappa, float(found)) == (float(c["result"][0]), float(c["result"][2])), c["name"]
    assert len(path) == (1 if path[0][1] else c["n_kappa"] + 1)


def _c2_transient():
    with np.load(GOLDEN.with_name("c2_transient.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("trial", range(16))
def test_c2_transient_grid_and_alg2_match_reference(orc, trial):
    """The oracle's grid step and Alg. 2 on the C2 transient-binding variant (1000
    scenarios, tests/golden/make_c2_transient_golden.py) equal the real reference's."""
    g = _c2_transient()
    n, js, m, nk = int(g["n_sim"]), int(g["j_star"]), int(g["m_grid"]), int(g["n_kappa"])
    rr = float(g["range"])
    x0, vp, r = g["x0"][trial], float(g["v_prev"][trial]), float(g["r"][trial])
    d = orc.sample(int(g["seed"][trial]), n, js + 1, [(-rr, rr)] * 3)
    tlo, thi = orc.tighten(-0.9, 0.9, 0.0, 0.05)
    k, v, f, _, P, st = orc.grid_step(0.01, x0, vp, r, m, d, -0.9, 0.9, tlo, thi, js,
                                      workers=orc.cpu_count())
    assert np.array_equal(np.packbits(P, axis=1), g["p_packed"][trial])
    assert [k, v, float(f)] == g["grid"][trial].tolist()
    assert [st["sims_run"], st["early_terms"], st["overflows"], st["ss_pruned_rows"],
            st["dedup_rows"]] == g["stats"][trial].tolist()
    ks, vs, fs, cells, early, _ = orc.robust_sequential(0.01, x0, vp, r, -0.9, 0.9, tlo, thi, d,
                                                        js, nk)
    assert [ks, vs, float(fs), cells, early] == g["seq"][trial].tolist()
    kj, fj, _ = orc.joint_bisect(0.01, x0, vp, r, -0.9, 0.9, tlo, thi, d, js, nk)
    assert (kj, float(fj)) == (ks, float(fs))
