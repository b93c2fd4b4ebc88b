"""Setpoint governors on the B200 (reference governor.py:1-579, drop-in names).

Same entry points, arguments, results and errors as the reference:

* ``robust_rg_parallel``   Alg. 3 grid search -> one fused kernel
  (csrc/rg_kernels.cu:k_grid): per-row steady-state gate and dedup, rollouts
  with the counter RNG fused in (or a staged tensor), warp-ballot feasibility
  reduction, extraction of the best row on the device.
* ``robust_rg_sequential`` Alg. 2 -> one kernel (k_bisect): every scenario runs
  its own bisection, then min / AND / sum reductions on the device.
* ``bisection_rg``         Alg. 1 -> the same kernel on the nominal prediction.
* ``fill_feasibility``     the full (candidate, scenario) matrix via the parity
  fill kernel (k_fill), with the reference's host-side gate, dedup and stats.

The numpy-tanh steady-state gate stays exactly the reference's: on the host
where the reference evaluates it per row (fill_feasibility), and on the device
as the verified setpoint interval of ssgate.py where the decision is made on
the device.  There is no CPU fallback: without the CUDA library or a device
every call raises BackendUnavailableError.
"""

from __future__ import annotations

import functools
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from .constraints import ConstraintSet, tighten, tighten_margin, validate_epsilon
from .disturbance import ScenarioSet
from .errors import BackendUnavailableError, ConfigError, DomainError, InfeasibleError, \
    RefgovError
from .ssgate import admissible_setpoints

__all__ = ["BACKENDS", "GovernorConfig", "GovernorState", "KappaResult", "CellProbe",
           "update_setpoint", "grid_kappas", "fill_feasibility", "extract_kappa_opt",
           "bisection_rg", "robust_rg_sequential", "robust_rg_parallel", "probe_candidate",
           "check_candidate", "DIAG_CSV_HEADER", "CELL_OK", "CELL_VIOLATED", "CELL_OVERFLOW",
           "robust_rg_parallel_batch", "robust_rg_joint"]

# "gpu" is the reference's name for its device backend (governor.py:53); both
# names select the CUDA device here.  CPU backends do not exist in this build.
BACKENDS = ("cuda", "gpu")
_POLICIES = ("hold", "error")
CELL_OK, CELL_VIOLATED, CELL_OVERFLOW = 1, 0, 2  # kernels.py:37-39

DIAG_CSV_HEADER = "t,kappa_opt,v,feasible,sims_run,early_terms,wall_us"


@dataclass
class GovernorConfig:
    """Governor knobs (governor.py:57-108) plus the device ones.

    device: CUDA ordinal.  keep_matrix: return the feasibility matrix P from
    robust_rg_parallel (the reference always does); False returns only the
    decision and lets rows already known infeasible stop early.
    ``workers`` is accepted for signature compatibility and ignored.
    """

    j_star: int = 256
    epsilon: float = 0.05
    n_kappa: int = 8
    m_grid: int = 32
    n_sim: int = 64
    backend: str = "cuda"
    infeasible_policy: str = "hold"
    prefix_mode: bool = False
    workers: int | None = None
    tighten_mode: str = "scale"
    device: int = 0
    keep_matrix: bool = True

    def __post_init__(self):
        if self.j_star < 1:
            raise ConfigError(f"j_star must be >= 1, got {self.j_star}")
        if self.tighten_mode == "scale":
            validate_epsilon(self.epsilon)
        elif self.tighten_mode == "margin":
            if not (np.isfinite(self.epsilon) and self.epsilon > 0):
                raise ConfigError(f"margin tightening needs epsilon > 0, got {self.epsilon}")
        else:
            raise ConfigError(f"tighten_mode must be scale or margin, got {self.tighten_mode!r}")
        if self.n_kappa < 1:
            raise ConfigError(f"n_kappa must be >= 1, got {self.n_kappa}")
        if self.m_grid < 2:
            raise ConfigError(f"m_grid must be >= 2, got {self.m_grid}")
        if self.n_sim < 1:
            raise ConfigError(f"n_sim must be >= 1, got {self.n_sim}")
        if self.backend not in BACKENDS:
            raise ConfigError(f"backend must be one of {BACKENDS}, got {self.backend!r}")
        if self.infeasible_policy not in _POLICIES:
            raise ConfigError(f"infeasible_policy must be one of {_POLICIES}, "
                              f"got {self.infeasible_policy!r}")
        if self.workers is not None and self.workers < 1:
            raise ConfigError(f"workers must be >= 1 or None, got {self.workers}")


@dataclass
class GovernorState:
    """The last applied setpoint, carried between timesteps."""

    v_prev: float = 0.0

    def __post_init__(self):
        if not math.isfinite(self.v_prev):
            raise ConfigError(f"v_prev must be finite, got {self.v_prev}")


@dataclass
class KappaResult:
    """Outcome of one governor call (governor.py:122-137)."""

    kappa_opt: float
    v_applied: float
    feasible: bool
    diagnostics: dict = field(default_factory=dict)
    matrix: np.ndarray | None = None

    def diagnostics_csv_row(self, t: int) -> str:
        d = self.diagnostics
        return (f"{t},{self.kappa_opt!r},{self.v_applied!r},{int(self.feasible)},"
                f"{d.get('sims_run', 0)},{d.get('early_terms', 0)},{d.get('wall_us', 0)}")


@dataclass(frozen=True)
class CellProbe:
    ok: bool
    steady_state_ok: bool
    status: int
    steps_run: int
    violation_step: int | None


def update_setpoint(v_prev: float, r: float, kappa: float) -> float:
    """v_prev + kappa (r - v_prev), exact at kappa = 0 and 1 (governor.py:151-159)."""
    if not 0.0 <= kappa <= 1.0:
        raise DomainError(f"kappa must lie in [0, 1], got {kappa}")
    if kappa == 0.0:
        return float(v_prev)
    if kappa == 1.0:
        return float(r)
    return float(v_prev + kappa * (r - v_prev))


def grid_kappas(m_grid: int) -> np.ndarray:
    """{i/(M-1)} ascending, endpoints exact (governor.py:162-166)."""
    if m_grid < 2:
        raise ConfigError(f"m_grid must be >= 2, got {m_grid}")
    return np.arange(m_grid, dtype=np.float64) / (m_grid - 1)


def extract_kappa_opt(P, prefix_mode: bool = False):
    """Best all-feasible row (1-based) and its kappa (governor.py:351-377)."""
    P = np.asarray(P)
    if P.ndim != 2 or P.size == 0:
        raise ConfigError(f"P must be a nonempty 2-D matrix, got shape {P.shape}")
    m = P.shape[0]
    full = P.all(axis=1)
    if prefix_mode:
        bad = np.flatnonzero(~full)
        idx = (int(bad[0]) if bad.size else m) - 1
    else:
        ok = np.flatnonzero(full)
        idx = int(ok[-1]) if ok.size else -1
    if idx < 0:
        return None, None
    if m == 1:
        return 1, 1.0
    return idx + 1, idx / (m - 1)


# ---------------------------------------------------------------------------
# host-side preparation shared by the entry points
# ---------------------------------------------------------------------------

def _tightened(cset, eps: float, mode: str) -> ConstraintSet:
    if mode == "scale":
        return tighten(cset, eps)
    if mode == "margin":
        return tighten_margin(cset, eps)
    raise ConfigError(f"tighten_mode must be scale or margin, got {mode!r}")


_DEVICE_KINDS = ("surrogate-fc", "linear")


def _require_device_plant(plant) -> str:
    kind = getattr(plant, "kernel_kind", None)
    if kind not in _DEVICE_KINDS:
        raise BackendUnavailableError(
            "the device kernels cover the surrogate fuel-cell plant and linear plants; "
            f"got plant kernel kind {kind!r}")
    return kind


def _require_surrogate(plant) -> None:
    if _require_device_plant(plant) != "surrogate-fc":
        raise BackendUnavailableError("this entry point is specialised to the surrogate plant")


def _validate_state(plant, x) -> np.ndarray:
    if hasattr(plant, "validate_state"):
        return plant.validate_state(x)
    n = int(getattr(plant, "state_dim", 3))
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (n,) or not np.all(np.isfinite(x)):
        raise ConfigError(f"state must be a finite vector of shape ({n},)")
    return x


def _problem(plant, cset, tight, j_star: int) -> _capi.Problem:
    v_lo, v_hi = admissible_setpoints(float(tight.lower), float(tight.upper))
    return _capi.Problem(float(plant.step_size), float(cset.lower), float(cset.upper), v_lo,
                         v_hi, int(j_star), 0)


def _source(scenarios, j_star: int, n_states: int = 3):
    """(dense tensor | None, n_sim, RNG stream | None) for the kernels.

    Mirrors _scenario_tensor (governor.py:169-179) for the shape checks.
    """
    if isinstance(scenarios, ScenarioSet) and scenarios.is_generated:
        if scenarios.state_dim != n_states:
            raise ConfigError(f"scenarios must be (n_sim, horizon, {n_states}), got state dim "
                              f"{scenarios.state_dim}")
        if scenarios.horizon < j_star + 1:
            raise ConfigError(f"scenario horizon {scenarios.horizon} too short: need >= "
                              f"j_star+1 = {j_star + 1}")
        if scenarios._stream is None:  # the rg_scenarios block is immutable: build it once
            scenarios._stream = _capi.make_scenarios(scenarios.seed, scenarios.k0,
                                                     scenarios.n_sim, scenarios.model.lo,
                                                     scenarios.model.span)
        return None, scenarios.n_sim, scenarios._stream
    data = scenarios.data if hasattr(scenarios, "data") else np.asarray(scenarios)
    data = np.asarray(data)
    if data.ndim != 3 or data.shape[2] != n_states:
        raise ConfigError(f"scenarios must be (n_sim, horizon, {n_states}), got {data.shape}")
    if data.shape[1] < j_star + 1:
        raise ConfigError(f"scenario horizon {data.shape[1]} too short: need >= "
                          f"j_star+1 = {j_star + 1}")
    if data.shape[0] < 1:
        raise ConfigError("need at least one scenario")
    return np.ascontiguousarray(data, dtype=np.float64), data.shape[0], None


def _host_rows(v_prev: float, r: float, grid, interval, gate=None):
    """v per row, the steady-state gate and the dedup map (governor.py:286, 302-317).

    The reference's own loop in Python floats (same three roundings as
    update_setpoint, endpoints exact), with the gate evaluated as the verified
    setpoint interval of ssgate.py -- identical to tight.contains(np.tanh(v))
    for every double -- and duplicates mapped to the first equal row through a
    dict, exactly as governor.py:306-317.  Returns Python lists.
    """
    d = r - v_prev
    v_rows = [v_prev if k == 0.0 else (r if k == 1.0 else v_prev + k * d) for k in grid]
    if gate is None:
        lo, hi = interval
        ss_ok = [lo <= v <= hi for v in v_rows]
    else:
        ss_ok = [gate(v) for v in v_rows]
    first: dict = {}
    dup_src = [-1] * len(v_rows)
    reps = []
    for i, v in enumerate(v_rows):
        if ss_ok[i]:
            j = first.get(v)
            if j is None:
                first[v] = i
                reps.append(i)
            else:
                dup_src[i] = j
    return v_rows, ss_ok, dup_src, reps


@functools.lru_cache(maxsize=256)
def _prepared(step_size, lower, upper, anchor, eps, mode, j_star, m_grid):
    """Per-configuration constants: the Problem block, the gate interval, the grid."""
    cset = ConstraintSet(lower, upper, anchor)
    tight = _tightened(cset, eps, mode)
    interval = admissible_setpoints(float(tight.lower), float(tight.upper))
    prob = _capi.Problem(float(step_size), float(lower), float(upper), interval[0],
                         interval[1], int(j_star), 0)
    grid = grid_kappas(m_grid) if m_grid else None
    return prob, interval, grid, (grid.tolist() if m_grid else None)


def _backend_check(backend: str) -> None:
    if backend not in BACKENDS:
        raise ConfigError(f"backend must be one of {BACKENDS}, got {backend!r}")


# ---------------------------------------------------------------------------
# fill_feasibility: the parity matrix
# ---------------------------------------------------------------------------

def fill_feasibility(backend, plant, x0, v_prev, r_t, grid, scenarios, cset, eps, j_star,
                     workers=None, stats=None, tighten_mode="scale", device: int = 0):
    """The (len(grid), n_sim) feasibility matrix P (governor.py:245-348).

    Every active (candidate, scenario) cell is one device thread; the
    steady-state gate, dedup and P assembly follow the reference line for line.
    """
    _backend_check(backend)
    grid = np.asarray(grid, dtype=np.float64)
    if grid.ndim != 1 or grid.size < 1:
        raise ConfigError(f"grid must be a nonempty 1-D array, got shape {grid.shape}")
    if np.any(np.diff(grid) < 0):
        raise ConfigError("grid must be sorted ascending")
    if np.any((grid < 0.0) | (grid > 1.0)) or not np.all(np.isfinite(grid)):
        raise ConfigError("grid entries must lie in [0, 1]")
    x0 = _validate_state(plant, x0)
    if tighten_mode == "scale":
        validate_epsilon(eps)
    if j_star < 1:
        raise ConfigError(f"j_star must be >= 1, got {j_star}")
    kind = _require_device_plant(plant)
    dist, n_sim, stream = _source(scenarios, j_star, int(plant.state_dim))
    tight = _tightened(cset, eps, tighten_mode)

    t0 = time.perf_counter()
    prob, interval, _, _ = _prepared(plant.step_size if kind == "surrogate-fc" else 1.0,
                                     cset.lower, cset.upper, cset.anchor, eps, tighten_mode,
                                     j_star, 0)
    gate = None if kind == "surrogate-fc" else (
        lambda v: tight.contains(plant.steady_state_output(v)))  # dc_gain * v (dynamics.py:199)
    v_rows, ss_ok, dup_src, rows = _host_rows(float(v_prev), float(r_t), grid.tolist(), interval,
                                              gate)
    v_rows = np.array(v_rows)
    ss_ok = np.array(ss_ok, dtype=bool)
    dup_src = np.array(dup_src, dtype=np.int64)
    rows = np.array(rows, dtype=np.int32)
    m = grid.size
    S = np.zeros((m, n_sim), dtype=np.uint8)
    steps = np.zeros((m, n_sim), dtype=np.int32)
    ctx = _capi.context(device)
    if kind == "surrogate-fc":
        ctx.fill(prob, x0, v_rows, rows, dist, n_sim, stream, S, steps)
    else:
        lin = _capi.make_linear(plant, tight.lower, tight.upper)
        ctx.fill_linear(lin, prob, x0, v_rows, rows, dist, n_sim, stream, S, steps)
    for i in np.flatnonzero(dup_src >= 0):
        S[i] = S[dup_src[i]]
        steps[i] = steps[dup_src[i]]
    P = (S == CELL_OK) & ss_ok[:, None]
    if stats is not None:
        ev = steps[rows] if rows.size else steps[:0]
        stats.update(
            backend="cuda", workers=1, device=ctx.device,
            sims_run=int(rows.size * n_sim),
            early_terms=int(np.count_nonzero(ev < j_star)),
            overflows=int(np.count_nonzero(S[rows] == CELL_OVERFLOW)) if rows.size else 0,
            ss_pruned_rows=int(np.count_nonzero(~ss_ok)),
            dedup_rows=int(np.count_nonzero(dup_src >= 0)),
            wall_us=int((time.perf_counter() - t0) * 1e6),
        )
    return P


# ---------------------------------------------------------------------------
# Alg. 3: robust grid step
# ---------------------------------------------------------------------------

def _robust_rg_parallel_via_fill(plant, x_t, state, r_t, cset, scenarios, config, backend):
    """governor.py:520-579 literally: fill the matrix, extract on the host (linear plants)."""
    grid = grid_kappas(config.m_grid)
    stats: dict = {}
    t0 = time.perf_counter()
    P = fill_feasibility(backend, plant, x_t, state.v_prev, r_t, grid, scenarios, cset,
                         config.epsilon, config.j_star, stats=stats,
                         tighten_mode=config.tighten_mode, device=getattr(config, "device", 0))
    row, _ = extract_kappa_opt(P, prefix_mode=config.prefix_mode)
    stats["wall_us"] = int((time.perf_counter() - t0) * 1e6)
    stats["method"] = "parallel-grid"
    if row is None:
        if config.infeasible_policy == "error":
            raise InfeasibleError("no candidate feasible, including kappa=0 (hold current "
                                  "setpoint)")
        return KappaResult(kappa_opt=0.0, v_applied=state.v_prev, feasible=False,
                           diagnostics=stats, matrix=P)
    kappa = float(grid[row - 1])
    v = update_setpoint(state.v_prev, r_t, kappa)
    state.v_prev = v
    return KappaResult(kappa_opt=kappa, v_applied=v, feasible=True, diagnostics=stats, matrix=P)


def robust_rg_parallel(plant, x_t, state, r_t, cset, scenarios, config, backend=None,
                       _matrix=None):
    """Scenario-robust governor step by grid search (governor.py:520-579).

    ``_matrix`` (internal): override config.keep_matrix for the matrix only -- False skips P
    but keeps every rollout to its end, so the diagnostics stay the reference's (the closed
    loop, which never reads P, uses it).
    """
    x_t = _validate_state(plant, x_t)
    backend = backend or config.backend
    _backend_check(backend)
    if _require_device_plant(plant) == "linear":
        return _robust_rg_parallel_via_fill(plant, x_t, state, r_t, cset, scenarios, config,
                                            backend)
    if config.tighten_mode == "scale":
        validate_epsilon(config.epsilon)
    prob, interval, grid, grid_list = _prepared(plant.step_size, cset.lower, cset.upper,
                                                cset.anchor, config.epsilon,
                                                config.tighten_mode, config.j_star,
                                                config.m_grid)
    dist, n_sim, stream = _source(scenarios, config.j_star)
    device = getattr(config, "device", 0)
    keep = getattr(config, "keep_matrix", True)

    t0 = time.perf_counter()
    ctx = _capi.context(device)
    want_p = keep if _matrix is None else bool(_matrix)
    res, viol, pbits = ctx.grid_step(prob, x_t, state.v_prev, r_t, config.m_grid,
                                     config.prefix_mode, dist, n_sim, stream, want_pbits=want_p,
                                     abandon=not keep, timing=False, want_viol=False)
    keep = want_p
    n_dup = 0
    # Without P (a closed loop) nothing below needs the host's row list, and the device's
    # gate/dedup counts came from the host's own plan (rg_capi.cu: episode_rows) anyway.
    if keep and (res.ss_pruned_rows or res.dedup_rows):
        # rows the device gated or deduplicated: the host's loop (governor.py:302-317)
        # names them, and must agree with the device's counts
        _, ss_ok, dup_src, _ = _host_rows(float(state.v_prev), float(r_t), grid_list, interval)
        n_pruned = ss_ok.count(False)
        n_dup = len(dup_src) - dup_src.count(-1)
        if res.ss_pruned_rows != n_pruned or res.dedup_rows != n_dup:
            raise RefgovError("device steady-state gate disagrees with the host gate")
    P = None
    if keep:
        # pruned and duplicate rows come back as zero bits; duplicates copy their source
        # (little-endian words: bit k % 32 of word k / 32 is byte-bit k % 8 of byte k / 8)
        P = np.unpackbits(pbits.view(np.uint8), axis=1, count=n_sim,
                          bitorder="little").view(np.bool_)
        if n_dup:
            for i, src in enumerate(dup_src):
                if src >= 0:
                    P[i] = P[src]
    row = None if res.row < 0 else res.row + 1
    stats = {"backend": "cuda", "workers": 1, "device": ctx.device, "sims_run": res.sims_run,
             "early_terms": res.early_terms, "overflows": res.overflows,
             "ss_pruned_rows": res.ss_pruned_rows, "dedup_rows": res.dedup_rows,
             "abandoned": res.abandoned, "kernel_us": int(res.kernel_ms * 1e3),
             "wall_us": int((time.perf_counter() - t0) * 1e6), "method": "parallel-grid"}
    if row is None:
        if config.infeasible_policy == "error":
            raise InfeasibleError("no candidate feasible, including kappa=0 (hold current "
                                  "setpoint)")
        return KappaResult(kappa_opt=0.0, v_applied=state.v_prev, feasible=False,
                           diagnostics=stats, matrix=P)
    kappa = float(grid[row - 1])
    v = update_setpoint(state.v_prev, r_t, kappa)
    state.v_prev = v
    return KappaResult(kappa_opt=kappa, v_applied=v, feasible=True, diagnostics=stats, matrix=P)


def robust_rg_parallel_batch(plant, X, v_prev, r, cset, model, n_sim, seeds, config, k0=0):
    """E independent robust grid steps in one device launch (BASELINE C3/C5).

    Episode e is robust_rg_parallel(plant, X[e], GovernorState(v_prev[e]), r[e],
    cset, sample_scenarios(model, n_sim, j_star+1, seeds[e]), config): returns
    (kappa[E], v_applied[E], feasible[E], early[E]), each equal to the
    single-episode call's result.  Under the "error" policy an episode with no
    feasible candidate raises InfeasibleError, as the single call does
    (governor.py:562-573).  Rows already known to be infeasible stop early
    (verdicts are unaffected).
    """
    _require_surrogate(plant)
    if config.tighten_mode == "scale":
        validate_epsilon(config.epsilon)
    X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, 3)
    if not np.all(np.isfinite(X)):
        raise ConfigError("state entries must be finite")
    if model.state_dim != 3 or model.kind != "uniform":
        raise ConfigError("the batched step needs a 3-state uniform disturbance model")
    prob, _, _, _ = _prepared(plant.step_size, cset.lower, cset.upper, cset.anchor,
                              config.epsilon, config.tighten_mode, config.j_star, 0)
    ctx = _capi.context(getattr(config, "device", 0))
    row, kappa, v, early = ctx.grid_step_batch(prob, X, v_prev, r, seeds, k0, n_sim, model.lo,
                                               model.span, config.m_grid, config.prefix_mode)
    if config.infeasible_policy == "error" and np.any(row < 0):
        bad = np.flatnonzero(row < 0)
        raise InfeasibleError(f"no candidate feasible, including kappa=0 (hold current "
                              f"setpoint), in episode(s) {bad[:8].tolist()}")
    return kappa, v, row >= 0, early


# ---------------------------------------------------------------------------
# Alg. 1 / Alg. 2: bisection
# ---------------------------------------------------------------------------

def _bisect_call(plant, x_t, state, r_t, cset, config, dist, n_sim, stream):
    kind = _require_device_plant(plant)
    prob, _, _, _ = _prepared(plant.step_size if kind == "surrogate-fc" else 1.0, cset.lower,
                              cset.upper, cset.anchor, config.epsilon, config.tighten_mode,
                              config.j_star, 0)
    ctx = _capi.context(getattr(config, "device", 0))
    if kind == "linear":
        tight = _tightened(cset, config.epsilon, config.tighten_mode)
        lin = _capi.make_linear(plant, tight.lower, tight.upper)
        res, _ = ctx.bisect_linear(lin, prob, x_t, state.v_prev, r_t, config.n_kappa, dist,
                                   n_sim, stream)
        return res
    res, _, _ = ctx.bisect(prob, x_t, state.v_prev, r_t, config.n_kappa, dist, n_sim, stream)
    return res


def bisection_rg(plant, x_t, state, r_t, cset, config):
    """Disturbance-free governor step by bisection (governor.py:433-466)."""
    x_t = _validate_state(plant, x_t)
    _require_device_plant(plant)
    t0 = time.perf_counter()
    res = _bisect_call(plant, x_t, state, r_t, cset, config, None, 1, None)
    kappa = float(res.kappa)
    v = update_setpoint(state.v_prev, r_t, kappa)
    state.v_prev = v
    return KappaResult(kappa_opt=kappa, v_applied=v, feasible=bool(res.found), diagnostics={
        "method": "bisection", "sims_run": int(res.cells), "early_terms": int(res.early),
        "kernel_us": int(res.kernel_ms * 1e3),
        "wall_us": int((time.perf_counter() - t0) * 1e6)})


def robust_rg_sequential(plant, x_t, state, r_t, cset, scenarios, config):
    """Worst case over per-scenario bisections (governor.py:469-517)."""
    x_t = _validate_state(plant, x_t)
    if scenarios.n_sim != config.n_sim:
        raise ConfigError(f"scenario count {scenarios.n_sim} does not match config.n_sim "
                          f"{config.n_sim}")
    _require_device_plant(plant)
    dist, n_sim, stream = _source(scenarios, config.j_star, int(plant.state_dim))
    t0 = time.perf_counter()
    res = _bisect_call(plant, x_t, state, r_t, cset, config, dist, n_sim, stream)
    kappa = float(res.kappa)
    v = update_setpoint(state.v_prev, r_t, kappa)
    state.v_prev = v
    return KappaResult(kappa_opt=kappa, v_applied=v, feasible=bool(res.found), diagnostics={
        "method": "sequential", "sims_run": int(res.cells), "early_terms": int(res.early),
        "kernel_us": int(res.kernel_ms * 1e3),
        "wall_us": int((time.perf_counter() - t0) * 1e6)})


def robust_rg_joint(plant, x_t, state, r_t, cset, scenarios, config):
    """Joint bisection: the scenario-robust step in the north-star form.

    The candidate sequence of _bisect_kappa (governor.py:407-431), each
    candidate tested on every scenario at once and feasible iff all stay inside
    the set; one device search (rg_bisect_joint) with an OR-reduced violation
    flag and early abandonment.  kappa_opt and feasible equal
    robust_rg_sequential's whenever every scenario's feasible set is a down-set
    in kappa; sims_run / early_terms count rollouts
    started and early terminations over all scenarios and iterations.
    """
    x_t = _validate_state(plant, x_t)
    if scenarios.n_sim != config.n_sim:
        raise ConfigError(f"scenario count {scenarios.n_sim} does not match config.n_sim "
                          f"{config.n_sim}")
    _require_surrogate(plant)
    dist, n_sim, stream = _source(scenarios, config.j_star)
    prob, _, _, _ = _prepared(plant.step_size, cset.lower, cset.upper, cset.anchor,
                              config.epsilon, config.tighten_mode, config.j_star, 0)
    t0 = time.perf_counter()
    ctx = _capi.context(getattr(config, "device", 0))
    res = ctx.bisect_joint(prob, x_t, state.v_prev, r_t, config.n_kappa, dist, n_sim, stream)
    kappa = float(res.kappa)
    v = update_setpoint(state.v_prev, r_t, kappa)
    state.v_prev = v
    return KappaResult(kappa_opt=kappa, v_applied=v, feasible=bool(res.found), diagnostics={
        "method": "joint", "sims_run": int(res.cells), "early_terms": int(res.early),
        "kernel_us": int(res.kernel_ms * 1e3),
        "wall_us": int((time.perf_counter() - t0) * 1e6)})


def bisect_paths(plant, x_t, v_prev, r_t, cset, scenarios, config):
    """Per-scenario bisection results and tested paths (parity diagnostics).

    Returns (kappa_k, found_k, cells_k, early_k, path_kappa, path_ok); unused
    path slots are NaN / 255.
    """
    x_t = _validate_state(plant, x_t)
    _require_surrogate(plant)
    dist, n_sim, stream = _source(scenarios, config.j_star)
    tight = _tightened(cset, config.epsilon, config.tighten_mode)
    ctx = _capi.context(getattr(config, "device", 0))
    prob = _problem(plant, cset, tight, config.j_star)
    _, per, paths = ctx.bisect(prob, x_t, v_prev, r_t, config.n_kappa, dist, n_sim, stream,
                               per_scenario=True, paths=True)
    return (*per, *paths)


# ---------------------------------------------------------------------------
# single-candidate diagnostics (governor.py:193-238)
# ---------------------------------------------------------------------------

def probe_candidate(plant, x0, v, scenario, cset, eps, j_star, tighten_mode="scale",
                    device: int = 0) -> CellProbe:
    x0 = _validate_state(plant, x0)
    n = int(plant.state_dim)
    scenario = np.asarray(scenario, dtype=np.float64)
    if scenario.ndim != 2 or scenario.shape[1] != n:
        raise ConfigError(f"scenario must be 2-D with {n} columns, got {scenario.shape}")
    if scenario.shape[0] < j_star + 1:
        raise ConfigError(f"scenario length {scenario.shape[0]} too short: need >= "
                          f"{j_star + 1}")
    kind = _require_device_plant(plant)
    tight = _tightened(cset, eps, tighten_mode)
    if not tight.contains(plant.steady_state_output(v)):
        return CellProbe(False, False, CELL_VIOLATED, 0, None)
    S = np.zeros((1, 1), dtype=np.uint8)
    steps = np.zeros((1, 1), dtype=np.int32)
    ctx = _capi.context(device)
    prob, _, _, _ = _prepared(plant.step_size if kind == "surrogate-fc" else 1.0, cset.lower,
                              cset.upper, cset.anchor, eps, tighten_mode, j_star, 0)
    args = (x0, np.array([float(v)]), np.array([0], np.int32), scenario[None], 1, None, S, steps)
    if kind == "linear":
        ctx.fill_linear(_capi.make_linear(plant, tight.lower, tight.upper), prob, *args)
    else:
        ctx.fill(prob, *args)
    st, sr = int(S[0, 0]), int(steps[0, 0])
    ok = st == CELL_OK
    return CellProbe(ok, True, st, sr, None if ok else sr)


def check_candidate(plant, x0, v, scenario, cset, eps, j_star, tighten_mode="scale") -> bool:
    return probe_candidate(plant, x0, v, scenario, cset, eps, j_star, tighten_mode).ok
