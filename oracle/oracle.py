"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the robust Reference Governor hot path.

This module restates the reference algorithm (arxiv 2510.08288, `refgov`
package, pkg/src/refgov) on the CPU so the CUDA product can be checked against
it on the GPU box, where /root/reference does not exist.  The per-cell rollout,
the fills and the scenario RNG run in C (rg_oracle.c, built by the Makefile
next to this file); the host-side governor logic is restated here in numpy.

Who may import this: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg -- as the checker or the timed CPU
baseline, never as the thing measured or shipped.  The product package
(paper_2510_08288_b200) never imports it.

Parity pinning: tests/test_oracle_golden.py compares every function here with
fixtures written by tests/golden/make_golden.py, which runs the real reference
(numba kernels, glibc libm tanh, numpy tanh) in the build container.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "librg_oracle.so"

CELL_OK, CELL_VIOLATED, CELL_OVERFLOW = 1, 0, 2  # kernels.py:37-39
STATE_LIMIT = 1e6  # kernels.py:42
_MASK = (1 << 64) - 1

_lib = None

_d = ctypes.c_double
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_p = ctypes.c_void_p


def build() -> Path:
    """Compile rg_oracle.c with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _SO


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not _SO.exists():
        build()
    L = ctypes.CDLL(str(_SO))
    L.orc_splitmix64.restype = _u64
    L.orc_splitmix64.argtypes = [_u64]
    L.orc_hash4.restype = _u64
    L.orc_hash4.argtypes = [_u64, _u64, _u64, _u64]
    L.orc_counter_uniform.restype = _d
    L.orc_counter_uniform.argtypes = [_u64, _u64, _u64, _u64]
    L.orc_sample.restype = None
    L.orc_sample.argtypes = [_u64, _i64, _i64, _i64, _i32, _p, _p, _p]
    L.orc_cell_sfc.restype = ctypes.c_int
    L.orc_cell_sfc.argtypes = [_d, _p, _d, _p, _i32, _d, _d, _p]
    L.orc_cell_sfc_rng.restype = ctypes.c_int
    L.orc_cell_sfc_rng.argtypes = [_d, _p, _d, _u64, _u64, _p, _p, _i32, _d, _d, _p]
    L.orc_fill_sfc.restype = ctypes.c_int
    L.orc_fill_sfc.argtypes = [_d, _p, _p, _p, _i64, _p, _i64, _i64, _i32, _d, _d, _p, _p,
                               _i32]
    L.orc_update_setpoint.restype = _d
    L.orc_update_setpoint.argtypes = [_d, _d, _d]
    L.orc_bisect_one.restype = _i32
    L.orc_bisect_one.argtypes = [_d, _p, _d, _d, _d, _d, _p, _i32, _i32, _d, _d, _p, _p, _p,
                                 _p, _p]
    L.orc_bisect_all.restype = None
    L.orc_bisect_all.argtypes = [_d, _p, _d, _d, _d, _d, _p, _i64, _i64, _i32, _i32, _d, _d,
                                 _p, _p, _p, _p]
    L.orc_cell_lin.restype = ctypes.c_int
    L.orc_cell_lin.argtypes = [_i32, _p, _p, _p, _d, _p, _d, _p, _i32, _d, _d, _p]
    L.orc_libm_tanh.restype = _d
    L.orc_libm_tanh.argtypes = [_d]
    L.orc_libm_tanh_many.restype = None
    L.orc_libm_tanh_many.argtypes = [_p, _p, _i64]
    _lib = L
    return L


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# RNG (disturbance.py:35-92, 179-203)
# --------------------------------------------------------------------------

def splitmix64(z: int) -> int:
    return int(lib().orc_splitmix64(z & _MASK))


def counter_uniform(seed: int, k: int, j: int, i: int) -> float:
    return float(lib().orc_counter_uniform(seed & _MASK, k & _MASK, j & _MASK, i & _MASK))


def derive_seed(master: int, label: str) -> int:
    """disturbance.py:64-69."""
    h = splitmix64(master & _MASK)
    for b in label.encode("utf-8"):
        h = splitmix64((h ^ b) & _MASK)
    return h


def sample(seed: int, n_sim: int, horizon: int, ranges, k0: int = 0) -> np.ndarray:
    """The (n_sim, horizon, n) tensor sample_scenarios returns (disturbance.py:179-203)."""
    ranges = [(float(a), float(b)) for a, b in ranges]
    lo = np.array([a for a, _ in ranges], dtype=np.float64)
    span = np.array([b - a for a, b in ranges], dtype=np.float64)
    out = np.empty((n_sim, horizon, len(ranges)), dtype=np.float64)
    lib().orc_sample(seed & _MASK, k0, n_sim, horizon, len(ranges), _ptr(lo), _ptr(span),
                     _ptr(out))
    return out


# --------------------------------------------------------------------------
# Cells and fills (kernels.py:47-86, 121-162, 260-313)
# --------------------------------------------------------------------------

def cell_sfc(h, x0, v, dist, n_steps, lo, hi):
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    dist = np.ascontiguousarray(dist, dtype=np.float64)
    sr = np.zeros(1, dtype=np.int32)
    st = lib().orc_cell_sfc(float(h), _ptr(x0), float(v), _ptr(dist), int(n_steps),
                            float(lo), float(hi), _ptr(sr))
    return int(st), int(sr[0])


def cell_sfc_rng(h, x0, v, seed, k, ranges, n_steps, lo, hi):
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    dlo = np.array([a for a, _ in ranges], dtype=np.float64)
    dspan = np.array([b - a for a, b in ranges], dtype=np.float64)
    sr = np.zeros(1, dtype=np.int32)
    st = lib().orc_cell_sfc_rng(float(h), _ptr(x0), float(v), seed & _MASK, k, _ptr(dlo),
                                _ptr(dspan), int(n_steps), float(lo), float(hi), _ptr(sr))
    return int(st), int(sr[0])


def run_cells(h, x0, v_rows, rows, dist, n_steps, lo, hi, S, steps, workers=1):
    """kernels.run_cells for the surrogate plant, writing S/steps in place."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    if rows.size == 0:
        return
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    v_rows = np.ascontiguousarray(v_rows, dtype=np.float64)
    dist = np.ascontiguousarray(dist, dtype=np.float64)
    assert S.flags.c_contiguous and steps.flags.c_contiguous
    rc = lib().orc_fill_sfc(float(h), _ptr(x0), _ptr(v_rows), _ptr(rows), rows.size,
                            _ptr(dist), dist.shape[0], dist.shape[1], int(n_steps),
                            float(lo), float(hi), _ptr(S), _ptr(steps), int(workers))
    if rc != 0:
        raise MemoryError("oracle fill allocation failed")


# --------------------------------------------------------------------------
# Governor host logic (governor.py:151-166, 245-377, 380-579)
# --------------------------------------------------------------------------

def update_setpoint(v_prev: float, r: float, kappa: float) -> float:
    """governor.py:151-159 (Python float arithmetic)."""
    if kappa == 0.0:
        return float(v_prev)
    if kappa == 1.0:
        return float(r)
    return float(v_prev + kappa * (r - v_prev))


def grid_kappas(m_grid: int) -> np.ndarray:
    """governor.py:162-166."""
    return np.arange(m_grid, dtype=np.float64) / (m_grid - 1)


def tighten(lower: float, upper: float, anchor: float, eps: float):
    """constraints.py:78-89 ("scale" mode)."""
    scale = 1.0 - eps
    lo = lower if np.isinf(lower) else anchor + scale * (lower - anchor)
    hi = upper if np.isinf(upper) else anchor + scale * (upper - anchor)
    return lo, hi


def ss_ok(v: float, tlo: float, thi: float) -> bool:
    """tight.contains(plant.steady_state_output(v)) with numpy's tanh (dynamics.py:243-244,
    constraints.py:62-66)."""
    y = float(np.tanh(v))
    if np.isnan(y):
        return False
    return tlo <= y <= thi


def fill_feasibility(h, x0, v_prev, r, grid, dist, lo, hi, tlo, thi, j_star, workers=1):
    """governor.py:245-348 for the serial/multicore backends.

    Returns (P, S, steps, stats) with the reference's stats keys (minus wall_us).
    """
    grid = np.asarray(grid, dtype=np.float64)
    m = grid.size
    n_sim = dist.shape[0]
    v_rows = np.array([update_setpoint(v_prev, r, float(k)) for k in grid])
    ok = np.array([ss_ok(v, tlo, thi) for v in v_rows])
    rep_for: dict = {}
    reps = []
    dup_src = np.full(m, -1, dtype=np.int64)
    for i in range(m):
        if not ok[i]:
            continue
        v = float(v_rows[i])
        if v in rep_for:
            dup_src[i] = rep_for[v]
        else:
            rep_for[v] = i
            reps.append(i)
    S = np.zeros((m, n_sim), dtype=np.uint8)
    steps = np.zeros((m, n_sim), dtype=np.int32)
    rows = np.array(reps, dtype=np.int64)
    run_cells(h, x0, v_rows, rows, dist, j_star, lo, hi, S, steps, workers=workers)
    for i in range(m):
        if dup_src[i] >= 0:
            S[i, :] = S[dup_src[i], :]
            steps[i, :] = steps[dup_src[i], :]
    P = (S == CELL_OK) & ok[:, None]
    evaluated = steps[rows, :] if rows.size else steps[:0, :]
    stats = dict(
        sims_run=int(rows.size * n_sim),
        early_terms=int(np.count_nonzero(evaluated < j_star)),
        overflows=int(np.count_nonzero(S[rows, :] == CELL_OVERFLOW)) if rows.size else 0,
        ss_pruned_rows=int(np.count_nonzero(~ok)),
        dedup_rows=int(np.count_nonzero(dup_src >= 0)),
    )
    return P, S, steps, stats


def extract_kappa_opt(P, prefix_mode=False):
    """governor.py:351-377."""
    P = np.asarray(P)
    m = P.shape[0]
    full = P.all(axis=1)
    if prefix_mode:
        idx = -1
        for i in range(m):
            if not full[i]:
                break
            idx = i
    else:
        idx = int(np.max(np.nonzero(full)[0])) if full.any() else -1
    if idx < 0:
        return None, None
    if m == 1:
        return 1, 1.0
    return idx + 1, idx / (m - 1)


def grid_step(h, x0, v_prev, r, m_grid, dist, lo, hi, tlo, thi, j_star, prefix_mode=False,
              workers=1):
    """robust_rg_parallel (governor.py:520-579), "hold" policy.

    Returns (kappa, v_applied, feasible, row, P, stats).
    """
    grid = grid_kappas(m_grid)
    P, _, _, stats = fill_feasibility(h, x0, v_prev, r, grid, dist, lo, hi, tlo, thi, j_star,
                                      workers)
    row, _ = extract_kappa_opt(P, prefix_mode)
    if row is None:
        return 0.0, float(v_prev), False, None, P, stats
    kappa = float(grid[row - 1])
    return kappa, update_setpoint(v_prev, r, kappa), True, row, P, stats


def bisect_kappa(h, x0, v_prev, r, lo, hi, tlo, thi, dist_k, j_star, n_kappa):
    """_bisect_kappa (governor.py:380-430) with the literal numpy-tanh gate.

    Returns (kappa, found, cells, early, path) where path lists (kappa, ok).
    """
    path = []

    def feasible_at(kappa):
        v = update_setpoint(v_prev, r, kappa)
        if not ss_ok(v, tlo, thi):
            return False, 0
        st, sr = cell_sfc(h, x0, v, dist_k, j_star, lo, hi)
        return st == CELL_OK, sr

    cells, early = 1, 0
    ok, sr = feasible_at(1.0)
    path.append((1.0, ok))
    if sr < j_star and not ok:
        early += 1
    if ok:
        return 1.0, True, cells, early, path
    klo, khi, kopt, found = 0.0, 1.0, 0.0, False
    for _ in range(n_kappa):
        kappa = 0.5 * (klo + khi)
        ok, sr = feasible_at(kappa)
        path.append((kappa, ok))
        cells += 1
        if sr < j_star and not ok:
            early += 1
        if ok:
            kopt, found, klo = kappa, True, kappa
        else:
            khi = kappa
    return kopt, found, cells, early, path


def robust_sequential(h, x0, v_prev, r, lo, hi, tlo, thi, dist, j_star, n_kappa):
    """robust_rg_sequential (governor.py:469-517).

    Returns (kappa, v_applied, feasible, cells, early, per_scenario) where
    per_scenario is a list of (kappa_k, found_k, cells_k, early_k, path_k).
    """
    kopt, feas, cells, early = 1.0, True, 0, 0
    per = []
    for k in range(dist.shape[0]):
        res = bisect_kappa(h, x0, v_prev, r, lo, hi, tlo, thi, dist[k], j_star, n_kappa)
        per.append(res)
        cells += res[2]
        early += res[3]
        feas = feas and res[1]
        kopt = min(kopt, res[0])
    return kopt, update_setpoint(v_prev, r, kopt), feas, cells, early, per


def joint_bisect(h, x0, v_prev, r, lo, hi, tlo, thi, dist, j_star, n_kappa, verdict=None):
    """Joint bisection: the candidate sequence of
    _bisect_kappa (governor.py:407-431), each candidate tested on every scenario
    at once and feasible iff all of them stay inside the set.

    ``verdict(v) -> (all_ok, n_early)`` may replace the scenario loop (the
    sharded tests pass a rank-local one and OR the flags).  Returns
    (kappa, found, path) with path = [(kappa, feasible), ...].
    """
    n = dist.shape[0]

    def default_verdict(v):
        ok_all, early = True, 0
        for k in range(n):
            st, sr = cell_sfc(h, x0, v, dist[k], j_star, lo, hi)
            ok_all &= st == CELL_OK
            early += int(st != CELL_OK and sr < j_star)
        return ok_all, early

    verdict = verdict or default_verdict
    path = []

    def feasible_at(kappa):
        v = update_setpoint(v_prev, r, kappa)
        if not ss_ok(v, tlo, thi):
            return False
        return verdict(v)[0]

    ok = feasible_at(1.0)
    path.append((1.0, ok))
    if ok:
        return 1.0, True, path
    klo, khi, kopt, found = 0.0, 1.0, 0.0, False
    for _ in range(n_kappa):
        kappa = 0.5 * (klo + khi)
        ok = feasible_at(kappa)
        path.append((kappa, ok))
        if ok:
            kopt, found, klo = kappa, True, kappa
        else:
            khi = kappa
    return kopt, found, path


def bisect_all_c(h, x0, v_prev, r, lo, hi, vlo, vhi, dist, j_star, n_kappa):
    """The same scenario loop in C with the steady-state gate given as the
    admissible setpoint interval [vlo, vhi] (for large N / CPU timing)."""
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    dist = np.ascontiguousarray(dist, dtype=np.float64)
    n = dist.shape[0]
    kap = np.empty(n)
    fnd = np.empty(n, dtype=np.int32)
    cel = np.empty(n, dtype=np.int32)
    erl = np.empty(n, dtype=np.int32)
    lib().orc_bisect_all(float(h), _ptr(x0), float(v_prev), float(r), float(vlo), float(vhi),
                         _ptr(dist), n, dist.shape[1], int(j_star), int(n_kappa), float(lo),
                         float(hi), _ptr(kap), _ptr(fnd), _ptr(cel), _ptr(erl))
    return kap, fnd, cel, erl


# --------------------------------------------------------------------------
# True plant and closed loops (dynamics.py:110-139, 209-244; harness.py:138-224)
# --------------------------------------------------------------------------

def _deriv(x, v):
    return np.array([-x[0] + np.tanh(x[1]), -x[1] + v, -2.0 * x[2] + x[0]], dtype=np.float64)


def plant_step(h, x, v):
    """rk4_step for the surrogate (dynamics.py:110-130, 228-231), numpy tanh.

    Returns None on the reference's IntegrationOverflowError condition.
    """
    k1 = _deriv(x, v)
    k2 = _deriv(x + 0.5 * h * k1, v)
    k3 = _deriv(x + 0.5 * h * k2, v)
    k4 = _deriv(x + h * k3, v)
    out = x + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    if np.any(~np.isfinite(out) | (np.abs(out) > STATE_LIMIT)):
        return None
    return out


def uniform_grid(seed, n_sim, horizon, width, k0=0):
    """_uniform_grid (disturbance.py:85-92) via the C hash."""
    out = sample(seed, n_sim, horizon, [(0.0, 1.0)] * width, k0=k0)
    return out


def closed_loop(h, lo, hi, anchor, eps, ranges, profile_sched, steps, seed, governor,
                n_sim=None, j_star=256, m_grid=32, n_kappa=8, x0=None, v0=0.0, workers=1):
    """run_closed_loop (harness.py:138-224) with a choice of governor.

    governor: "grid" (robust_rg_parallel, the reference driver) or "bisection"
    (bisection_rg substituted at harness.py:200, configuration C1).
    Returns a list of (t, r_t, v_t, y_t, kappa, feasible) rows and an abort flag.
    """
    tlo, thi = tighten(lo, hi, anchor, eps)
    x = np.zeros(3) if x0 is None else np.asarray(x0, dtype=np.float64)
    v_prev = float(v0)
    scen_seed = derive_seed(seed, "scenarios")
    plant_seed = derive_seed(seed, "plant")
    rlo = np.array([a for a, _ in ranges])
    span = np.array([b - a for a, b in ranges])
    d_true = rlo + span * uniform_grid(plant_seed, 1, steps, 3)[0]
    rows = []
    zero = np.zeros((j_star + 1, 3))
    for t in range(steps):
        r_t = float(profile_sched[t])
        if governor == "grid":
            dist = sample((scen_seed + t) & _MASK, n_sim, j_star + 1, ranges)
            kappa, v_t, feas, _, _, _ = grid_step(h, x, v_prev, r_t, m_grid, dist, lo, hi,
                                                  tlo, thi, j_star, workers=workers)
        else:
            kappa, feas, _, _, _ = bisect_kappa(h, x, v_prev, r_t, lo, hi, tlo, thi, zero,
                                                j_star, n_kappa)
            v_t = update_setpoint(v_prev, r_t, kappa)
        v_prev = v_t
        y_t = float(x[0])
        rows.append((t, r_t, v_t, y_t, float(kappa), bool(feas)))
        nx = plant_step(h, x, v_t)
        if nx is None:
            return rows, True
        x = nx + d_true[t]
        if not np.all(np.isfinite(x)) or np.any(np.abs(x) > STATE_LIMIT):
            return rows, True
    return rows, False


def profile_schedule(points, steps):
    """ReferenceProfile.schedule (harness.py:80-89)."""
    out = np.empty(steps)
    idx = 0
    r = float(points[0][1])
    for t in range(steps):
        while idx < len(points) and points[idx][0] <= t:
            r = float(points[idx][1])
            idx += 1
        out[t] = r
    return out


# --------------------------------------------------------------------------
# Linear plant (kernels.py:90-118; dynamics.py:162-206; governor.py paths)
# --------------------------------------------------------------------------

def cell_lin(A, B, C, D, x0, v, dist, n_steps, lo, hi):
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    C = np.ascontiguousarray(C, dtype=np.float64)
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    dist = np.ascontiguousarray(dist, dtype=np.float64)
    sr = np.zeros(1, dtype=np.int32)
    st = lib().orc_cell_lin(int(x0.size), _ptr(A), _ptr(B), _ptr(C), float(D), _ptr(x0),
                            float(v), _ptr(dist), int(n_steps), float(lo), float(hi), _ptr(sr))
    return int(st), int(sr[0])


def fill_feasibility_lin(A, B, C, D, dc_gain, x0, v_prev, r, grid, dist, lo, hi, tlo, thi,
                         j_star):
    """governor.py:245-348 for a LinearOraclePlant (gate: tight.contains(dc_gain * v))."""
    grid = np.asarray(grid, dtype=np.float64)
    m, n_sim = grid.size, dist.shape[0]
    v_rows = [update_setpoint(v_prev, r, float(k)) for k in grid]
    ok = np.array([tlo <= dc_gain * v <= thi for v in v_rows])
    first, reps, dup = {}, [], np.full(m, -1)
    for i in range(m):
        if ok[i]:
            if v_rows[i] in first:
                dup[i] = first[v_rows[i]]
            else:
                first[v_rows[i]] = i
                reps.append(i)
    S = np.zeros((m, n_sim), dtype=np.uint8)
    steps = np.zeros((m, n_sim), dtype=np.int32)
    for i in reps:
        for k in range(n_sim):
            S[i, k], steps[i, k] = cell_lin(A, B, C, D, x0, v_rows[i], dist[k], j_star, lo, hi)
    for i in range(m):
        if dup[i] >= 0:
            S[i], steps[i] = S[dup[i]], steps[dup[i]]
    P = (S == CELL_OK) & ok[:, None]
    return P, S, steps


def bisect_kappa_lin(A, B, C, D, dc_gain, x0, v_prev, r, lo, hi, tlo, thi, dist_k, j_star,
                     n_kappa):
    """_bisect_kappa (governor.py:380-430) for a LinearOraclePlant."""
    def feasible_at(kappa):
        v = update_setpoint(v_prev, r, kappa)
        if not tlo <= dc_gain * v <= thi:
            return False, 0
        st, sr = cell_lin(A, B, C, D, x0, v, dist_k, j_star, lo, hi)
        return st == CELL_OK, sr

    cells, early = 1, 0
    ok, sr = feasible_at(1.0)
    if sr < j_star and not ok:
        early += 1
    if ok:
        return 1.0, True, cells, early
    klo, khi, kopt, found = 0.0, 1.0, 0.0, False
    for _ in range(n_kappa):
        kappa = 0.5 * (klo + khi)
        ok, sr = feasible_at(kappa)
        cells += 1
        if sr < j_star and not ok:
            early += 1
        if ok:
            kopt, found, klo = kappa, True, kappa
        else:
            khi = kappa
    return kopt, found, cells, early


def linear_maximal_kappa(A, B, C, D, x0, v_prev, r, lower, upper, tlo, thi, j_star,
                         resolution=1_000_001):
    """oracle.py:115-198 of the reference: the exact maximal kappa of a stable
    linear plant on the nominal prediction, snapped to a 10^6-point grid.

    y_j = c_j + g_j v with c_j = C A^j x0 and g_j = C sum_{l<j} A^l B + D; each
    bound at each step admits a closed-form kappa interval.
    """
    A = np.atleast_2d(np.asarray(A, dtype=np.float64))
    B = np.asarray(B, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    n = A.shape[0]
    gain = float(C @ np.linalg.solve(np.eye(n) - A, B) + D)
    c = np.empty(j_star + 1)
    g = np.empty(j_star + 1)
    alpha = np.asarray(x0, dtype=np.float64).copy()
    beta = np.zeros(n)
    for j in range(j_star + 1):
        c[j] = float(C @ alpha)
        g[j] = float(C @ beta) + D
        alpha = A @ alpha
        beta = A @ beta + B
    delta = r - v_prev
    lo_k, hi_k = 0.0, 1.0

    def clamp(p, q, lo, hi):
        nonlocal lo_k, hi_k
        if q == 0.0:
            return lo <= p <= hi
        a, b = (lo - p) / q, (hi - p) / q
        if a > b:
            a, b = b, a
        lo_k, hi_k = max(lo_k, a), min(hi_k, b)
        return True

    for j in range(j_star + 1):
        if not clamp(c[j] + g[j] * v_prev, g[j] * delta, lower, upper):
            return None
    if not clamp(gain * v_prev, gain * delta, tlo, thi) or lo_k > hi_k:
        return None

    def ok_at(kappa):
        v = update_setpoint(v_prev, r, kappa)
        y = c + g * v
        return bool(np.all(y >= lower) and np.all(y <= upper) and tlo <= gain * v <= thi)

    i = min(resolution - 1, int(np.floor(hi_k * (resolution - 1) + 1e-12)))
    for _ in range(4):
        if i < 0:
            return None
        kappa = i / (resolution - 1)
        if ok_at(kappa):
            return float(kappa)
        i -= 1
    return None


def libm_tanh(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    lib().orc_libm_tanh_many(_ptr(x), _ptr(y), x.size)
    return y


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
