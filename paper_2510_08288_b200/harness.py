"""Closed-loop drivers (reference harness.py:52-224), governor on the B200.

``run_closed_loop`` is the reference's driver with the device grid governor:
every step the scenario set is the counter stream ``derive_seed(seed,
"scenarios") + t`` (generated inside the kernel, never materialised), the
governor picks v_t, and the true plant advances on the host with numpy's tanh
plus its own disturbance stream ``derive_seed(seed, "plant")`` -- exactly the
reference's arithmetic, so the v_t sequence is bit-identical.

The governed loop runs in the library by default (``rg_closed_loop``: the grid step,
kappa and v_t, and the true plant's RK4 step with the library's restatement of numpy's
tanh, without a Python round trip; the whole trace as one device kernel, k_loop_ts, or
with the "no_device_loop" option one grid-step launch per step and the plant in C on the
host); ``native=False`` keeps the per-step Python loop below, which the tests hold both to
bit for bit.

``run_closed_loop_bisection`` substitutes the nominal ``bisection_rg`` at
harness.py:200 (configuration C1 of BASELINE.md; the reference ships no such
driver).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .disturbance import DisturbanceModel, ScenarioSet, derive_seed, sample_scenarios
from .errors import ConfigError, InfeasibleError, IntegrationOverflowError
from .governor import GovernorState, bisection_rg, robust_rg_parallel, \
    robust_rg_parallel_batch

__all__ = ["ReferenceProfile", "RunRecord", "TimingRecord", "run_closed_loop",
           "run_closed_loop_bisection", "run_closed_loop_batch", "bench_sweep",
           "parse_nsim_spec", "emit_csv", "RUN_CSV_HEADER", "TIMING_CSV_HEADER", "STATE_LIMIT"]

RUN_CSV_HEADER = "t,r_t,v_t,y_t,kappa_opt,feasible,wall_us"
TIMING_CSV_HEADER = "backend,n_sim,mode,mean_us,min_us,max_us,reps"
_BENCH_MODES = ("kernel-only", "end-to-end")
STATE_LIMIT = 1e6


@dataclass(frozen=True)
class ReferenceProfile:
    """Piecewise-constant reference r(t) from (t_start, r) points (harness.py:52-89)."""

    points: tuple

    def __post_init__(self):
        try:
            pts = tuple((int(t), float(r)) for t, r in self.points)
        except (TypeError, ValueError) as e:
            raise ConfigError(f"profile points must be (t_start, r) pairs: {e}") from None
        if not pts:
            raise ConfigError("profile needs at least one (t_start, r) point")
        if pts[0][0] != 0:
            raise ConfigError(f"first profile point must start at t=0, got {pts[0][0]}")
        if any(b[0] <= a[0] for a, b in zip(pts, pts[1:])):
            raise ConfigError("profile t_start values must be strictly increasing")
        object.__setattr__(self, "points", pts)

    def schedule(self, steps: int) -> np.ndarray:
        starts = np.array([t for t, _ in self.points])
        vals = np.array([r for _, r in self.points])
        idx = np.searchsorted(starts, np.arange(steps), side="right") - 1
        return vals[idx]


@dataclass
class RunRecord:
    rows: list
    config: dict
    seed: int
    aborted: bool = False
    abort_reason: str | None = None
    diag_rows: list = field(default_factory=list)

    def violations(self, cset) -> int:
        return sum(1 for row in self.rows if not cset.contains(row[3]))


def _true_disturbance(model: DisturbanceModel, steps: int, seed: int, device: int) -> np.ndarray:
    # lo + span * u at (plant_seed, 0, t, i): harness.py:172-174
    return sample_scenarios(model, 1, steps, derive_seed(seed, "plant"), device=device).data[0]


def _schedule(profile, steps):
    if isinstance(profile, ReferenceProfile):
        return profile.schedule(steps)
    return np.asarray(profile, dtype=np.float64)[:steps]


_NP_TANH_PROBE: list = []


def _np_tanh_matches() -> bool:
    """Whether the library's restatement of numpy's tanh (rg_nptanh.h: numpy's AVX512/AVX2
    kernel) is this process's np.tanh -- checked once on values across every interval and
    its boundaries.  A numpy without that kernel (no AVX2 on the host: libm's tanh) keeps
    the closed loop's true plant in Python, where it calls np.tanh itself."""
    if not _NP_TANH_PROBE:
        from . import _capi

        rng = np.random.default_rng(1)
        edges = np.array([0.1875 * 2.0 ** e * m for e in range(-3, 7) for m in (1.0, 1.5)])
        near = (edges[:, None].view(np.int64) + np.arange(-8, 9)[None, :]).ravel()
        x = np.concatenate([rng.uniform(-30, 30, 2048), rng.uniform(-1, 1, 2048),
                            near.view(np.float64), -near.view(np.float64)])
        ok = np.array_equal(_capi.np_tanh(x).view(np.uint64), np.tanh(x).view(np.uint64))
        _NP_TANH_PROBE.append(bool(ok))
    return _NP_TANH_PROBE[0]


def _native_loop_ok(plant, config, grid=True) -> bool:
    from .dynamics import SurrogateFuelCellPlant

    return (type(plant) is SurrogateFuelCellPlant and getattr(config, "backend", "cuda") == "cuda"
            and (not grid or bool(getattr(config, "m_grid", 0))) and _np_tanh_matches())


def _run_closed_loop_bisection_native(plant, cset, model, config, profile, steps, seed, x0, v0):
    """run_closed_loop_bisection through rg_closed_loop_bisection: the same plant stream,
    the same bisection (governor.py:380-430 with zero disturbance), update_setpoint and
    true-plant arithmetic, the same KappaResults; the plant's integration overflow raises as
    plant.step does."""
    from . import _capi
    from .governor import KappaResult, _prepared

    if steps < 1:
        raise ConfigError(f"steps must be >= 1, got {steps}")
    device = getattr(config, "device", 0)
    x = plant.validate_state(np.zeros(plant.state_dim) if x0 is None else x0)
    prob = _prepared(plant.step_size, cset.lower, cset.upper, cset.anchor, config.epsilon,
                     config.tighten_mode, config.j_star, 0)[0]
    d_true = _true_disturbance(model, steps, seed, device)
    r_sched = np.ascontiguousarray(_schedule(profile, steps), dtype=np.float64)
    if r_sched.size < steps:
        raise ConfigError(f"profile has {r_sched.size} entries, need {steps}")
    ctx = _capi.context(device)
    res, out, _ = ctx.closed_loop_bisection(prob, config.n_kappa, x, float(v0), r_sched[:steps],
                                            d_true)
    if res.abort_kind == _capi.RG_LOOP_OVERFLOW:
        raise IntegrationOverflowError(f"integration overflow in state {res.abort_index} "
                                       f"(value {np.float64(res.abort_value)!r})",
                                       state_index=res.abort_index)
    k_l, v_l, y_l = out["kappa"].tolist(), out["v"].tolist(), out["y"].tolist()
    f_l, c_l, e_l, w_l = (out["found"].tolist(), out["cells"].tolist(), out["early"].tolist(),
                          out["wall_us"].tolist())
    return [(KappaResult(kappa_opt=k_l[t], v_applied=v_l[t], feasible=bool(f_l[t]),
                         diagnostics={"method": "bisection", "sims_run": c_l[t],
                                      "early_terms": e_l[t], "kernel_us": w_l[t],
                                      "wall_us": w_l[t]}), y_l[t])
            for t in range(res.steps_done)]


def _run_closed_loop_native(plant, cset, model, config, profile, steps, seed, x0, v0):
    """run_closed_loop's governed loop through rg_closed_loop: the same scenario and plant
    streams, the same device step, kappa, update_setpoint and true-plant arithmetic (numpy's
    tanh restated, rg_nptanh.h), the same rows, diagnostics and abort reasons."""
    from . import _capi
    from .governor import _prepared, validate_epsilon

    device = getattr(config, "device", 0)
    x = plant.validate_state(np.zeros(plant.state_dim) if x0 is None else x0)
    if config.tighten_mode == "scale":
        validate_epsilon(config.epsilon)
    prob = _prepared(plant.step_size, cset.lower, cset.upper, cset.anchor, config.epsilon,
                     config.tighten_mode, config.j_star, config.m_grid)[0]
    scen_seed = derive_seed(seed, "scenarios")
    d_true = _true_disturbance(model, steps, seed, device)
    r_sched = np.ascontiguousarray(_schedule(profile, steps), dtype=np.float64)
    if r_sched.size < steps:
        raise ConfigError(f"profile has {r_sched.size} entries, need {steps}")
    ctx = _capi.context(device)
    res, out, _ = ctx.closed_loop(prob, config.m_grid, config.prefix_mode,
                                  config.infeasible_policy == "error", x, float(v0),
                                  r_sched[:steps], d_true, scen_seed, config.n_sim, model.lo,
                                  model.span)
    rec = RunRecord(rows=[], config={"governor_on": True, "j_star": config.j_star,
                                     "n_sim": config.n_sim, "m_grid": config.m_grid,
                                     "steps": steps, "backend": "cuda"}, seed=seed)
    r_l, v_l, y_l = r_sched.tolist(), out["v"].tolist(), out["y"].tolist()
    k_l, f_l, w_l = out["kappa"].tolist(), out["feasible"].tolist(), out["wall_us"].tolist()
    s_l, e_l = out["sims_run"].tolist(), out["early_terms"].tolist()
    for t in range(res.steps_done):
        feas = bool(f_l[t])
        rec.rows.append((t, r_l[t], v_l[t], y_l[t], k_l[t], feas, w_l[t]))
        rec.diag_rows.append(f"{t},{k_l[t]!r},{v_l[t]!r},{int(feas)},{s_l[t]},{e_l[t]},{w_l[t]}")
    if res.abort_kind == _capi.RG_LOOP_INFEASIBLE:
        raise InfeasibleError("no candidate feasible, including kappa=0 (hold current setpoint)")
    if res.abort_kind == _capi.RG_LOOP_OVERFLOW:
        # the Python plant reports the numpy scalar (dynamics.py: _surrogate_rk4)
        e = IntegrationOverflowError(f"integration overflow in state {res.abort_index} "
                                     f"(value {np.float64(res.abort_value)!r})",
                                     state_index=res.abort_index)
        rec.aborted, rec.abort_reason = True, f"step {res.abort_step}: {e}"
    elif res.abort_kind == _capi.RG_LOOP_LEFT_BOX:
        rec.aborted = True
        rec.abort_reason = f"step {res.abort_step}: state left the operating box"
    return rec


def run_closed_loop(plant, cset, model, config, profile, steps, seed, governor_on=True,
                    x0=None, v0=0.0, native=None) -> RunRecord:
    """The governed closed loop of harness.py:138-224 with the device governor.

    ``native`` (default: whenever the plant is the surrogate and the governor is on): the
    loop runs in the library (rg_closed_loop) instead of step by step in Python.
    """
    if steps < 1:
        raise ConfigError(f"steps must be >= 1, got {steps}")
    if model.state_dim != plant.state_dim:
        raise ConfigError(f"disturbance model has {model.state_dim} states, plant has "
                          f"{plant.state_dim}")
    if native is None:
        native = governor_on and _native_loop_ok(plant, config)
    if native:
        if not governor_on:
            raise ConfigError("the native closed loop runs the governor")
        return _run_closed_loop_native(plant, cset, model, config, profile, steps, seed, x0, v0)
    device = getattr(config, "device", 0)
    x = plant.validate_state(np.zeros(plant.state_dim) if x0 is None else x0)
    state = GovernorState(v_prev=float(v0))
    scen_seed = derive_seed(seed, "scenarios")
    d_true = _true_disturbance(model, steps, seed, device)
    r_sched = _schedule(profile, steps)
    rec = RunRecord(rows=[], config={"governor_on": governor_on, "j_star": config.j_star,
                                     "n_sim": config.n_sim, "m_grid": config.m_grid,
                                     "steps": steps, "backend": "cuda"}, seed=seed)
    for t in range(steps):
        r_t = float(r_sched[t])
        if governor_on:
            scen = sample_scenarios(model, config.n_sim, config.j_star + 1, seed=scen_seed + t,
                                    device=device)
            t0 = time.perf_counter()
            # the loop never reads P: skip it, keep the reference's diagnostics
            res = robust_rg_parallel(plant, x, state, r_t, cset, scen, config, _matrix=False)
            wall_us = int((time.perf_counter() - t0) * 1e6)
            v_t, kappa, feas = res.v_applied, res.kappa_opt, res.feasible
            rec.diag_rows.append(res.diagnostics_csv_row(t))
        else:
            v_t, kappa, feas, wall_us = r_t, 1.0, True, 0
            state.v_prev = v_t
        rec.rows.append((t, r_t, v_t, float(plant.output(x, v_t)), float(kappa), bool(feas),
                         wall_us))
        try:
            x = plant.step(x, v_t) + d_true[t]
        except IntegrationOverflowError as e:
            rec.aborted, rec.abort_reason = True, f"step {t}: {e}"
            return rec
        if not np.all(np.isfinite(x)) or np.any(np.abs(x) > STATE_LIMIT):
            rec.aborted, rec.abort_reason = True, f"step {t}: state left the operating box"
            return rec
    return rec


def run_closed_loop_bisection(plant, cset, model, config, profile, steps, seed, x0=None,
                              v0=0.0, native=None):
    """C1: the same loop with the nominal bisection governor; returns
    [(KappaResult, y_t)] per step.

    ``native`` (default: for the surrogate plant when the library's numpy tanh is this
    process's): the whole loop runs on the device as one kernel (rg_closed_loop_bisection:
    the bisection's candidates on the time-split passes, the true plant with numpy's tanh
    restated); ``native=False`` keeps the per-step loop over bisection_rg below, which the
    tests hold it to bit for bit.  ``wall_us`` is then each step's device time.
    """
    if native is None:
        native = _native_loop_ok(plant, config, grid=False)
    if native:
        return _run_closed_loop_bisection_native(plant, cset, model, config, profile, steps,
                                                 seed, x0, v0)
    device = getattr(config, "device", 0)
    x = plant.validate_state(np.zeros(plant.state_dim) if x0 is None else x0)
    state = GovernorState(v_prev=float(v0))
    d_true = _true_disturbance(model, steps, seed, device)
    r_sched = _schedule(profile, steps)
    out = []
    for t in range(steps):
        y_t = float(plant.output(x, state.v_prev))
        res = bisection_rg(plant, x, state, float(r_sched[t]), cset, config)
        out.append((res, y_t))
        x = plant.step(x, res.v_applied) + d_true[t]
    return out


def _rk4_batch(h: float, X: np.ndarray, V: np.ndarray) -> np.ndarray:
    """The surrogate's rk4_step on E states at once (dynamics.py:110-139).

    Elementwise the same IEEE operations as the scalar step; numpy's vector
    and scalar tanh agree bit for bit (tests/test_harness_batch.py).
    """
    def f(Y):
        out = np.empty_like(Y)
        out[:, 0] = -Y[:, 0] + np.tanh(Y[:, 1])
        out[:, 1] = -Y[:, 1] + V
        out[:, 2] = -2.0 * Y[:, 2] + Y[:, 0]
        return out

    k1 = f(X)
    k2 = f(X + 0.5 * h * k1)
    k3 = f(X + 0.5 * h * k2)
    k4 = f(X + h * k3)
    return X + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


def run_closed_loop_batch(plant, cset, model, config, profile, steps, seeds, x0=None, v0=0.0,
                          devices=None):
    """E independent governed closed loops (BASELINE C5), one device launch per step.

    Episode e is run_closed_loop(plant, cset, model, config, profile, steps,
    seeds[e]) -- same scenario and plant streams, same arithmetic -- with all
    live episodes' governor steps batched into rg_grid_step_batch and the true
    plants advanced together with numpy.  `profile` is one profile for all
    episodes or an (E, steps) array of requests.  `devices` (default: config.device)
    spreads the episodes over several GPUs as replicas: contiguous episode ranges, one
    batched launch per device per step, the devices' calls issued concurrently from
    host threads (each device has its own context and stream; the C calls release the
    GIL).  Returns one RunRecord per episode (rows: t, r_t, v_t, y_t, kappa, feasible,
    wall_us=0).
    """
    import dataclasses
    from concurrent.futures import ThreadPoolExecutor

    seeds = [int(s_) for s_ in seeds]
    E = len(seeds)
    if steps < 1 or E < 1:
        raise ConfigError("steps and the number of episodes must be >= 1")
    devices = [getattr(config, "device", 0)] if devices is None else [int(d) for d in devices]
    if not devices:
        raise ConfigError("devices must be nonempty")
    device = devices[0]
    X = np.tile(np.zeros(3) if x0 is None else np.asarray(x0, dtype=np.float64), (E, 1))
    Vp = np.full(E, float(v0))
    if isinstance(profile, ReferenceProfile):
        R = np.tile(profile.schedule(steps), (E, 1))
    else:
        R = np.asarray(profile, dtype=np.float64).reshape(E, -1)[:, :steps]
    scen_seeds = np.array([derive_seed(s_, "scenarios") for s_ in seeds], dtype=object)
    D = np.stack([_true_disturbance(model, steps, s_, device) for s_ in seeds])
    recs = [RunRecord(rows=[], config={"j_star": config.j_star, "n_sim": config.n_sim,
                                       "m_grid": config.m_grid, "steps": steps,
                                       "backend": "cuda", "batched": E,
                                       "devices": list(devices)}, seed=s_)
            for s_ in seeds]
    # episode e runs on devices[owner[e]]: contiguous ranges, as even as possible
    owner = (np.arange(E) * len(devices)) // E
    cfgs = [dataclasses.replace(config, device=d) for d in devices]
    pool = ThreadPoolExecutor(len(devices)) if len(devices) > 1 else None
    live = np.arange(E)

    def governor(q, idx, t):
        return robust_rg_parallel_batch(plant, X[idx], Vp[idx], R[idx, t], cset, model,
                                        config.n_sim, [(int(scen_seeds[e]) + t) for e in idx],
                                        cfgs[q])

    try:
        for t in range(steps):
            if live.size == 0:
                break
            parts = [live[owner[live] == q] for q in range(len(devices))]
            jobs = [(q, idx) for q, idx in enumerate(parts) if idx.size]
            if pool is None:
                outs = [governor(q, idx, t) for q, idx in jobs]
            else:
                outs = list(pool.map(lambda j: governor(j[0], j[1], t), jobs))
            kap = np.empty(live.size)
            v = np.empty(live.size)
            feas = np.empty(live.size, dtype=bool)
            pos = {e: j for j, e in enumerate(live)}
            for (q, idx), (k_, v_, f_, _) in zip(jobs, outs):
                at = np.array([pos[e] for e in idx])
                kap[at], v[at], feas[at] = k_, v_, f_
            for j, e in enumerate(live):
                recs[e].rows.append((t, float(R[e, t]), float(v[j]), float(X[e, 0]),
                                     float(kap[j]), bool(feas[j]), 0))
            Vp[live] = v
            Xn = _rk4_batch(plant.step_size, X[live], v)
            bad = np.any(~np.isfinite(Xn) | (np.abs(Xn) > STATE_LIMIT), axis=1)
            Xn = Xn + D[live, t]
            bad2 = np.any(~np.isfinite(Xn) | (np.abs(Xn) > STATE_LIMIT), axis=1)
            X[live] = Xn
            for j in np.flatnonzero(bad | bad2):
                e = live[j]
                recs[e].aborted = True
                recs[e].abort_reason = (f"step {t}: integration overflow" if bad[j] else
                                        f"step {t}: state left the operating box")
            live = live[~(bad | bad2)]
    finally:
        if pool is not None:
            pool.shutdown()
    return recs


# ---------------------------------------------------------------------------
# Benchmark sweep and CSV emission (harness.py:114-136, 227-414): the
# reference's measurement API, so its timing CSVs come out of the device path.
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class TimingRecord:
    """One (backend, n_sim, mode) timing summary (harness.py:114-136)."""

    backend: str
    n_sim: int
    m_grid: int
    reps: int
    mode: str
    mean_us: float | None
    min_us: float | None
    max_us: float | None
    skipped: bool = False

    def __post_init__(self):
        if not self.skipped:
            if self.reps < 1:
                raise ConfigError(f"reps must be >= 1, got {self.reps}")
            if not (self.min_us <= self.mean_us <= self.max_us):
                raise ConfigError("mean outside [min, max]")


def parse_nsim_spec(spec: str) -> list[int]:
    """"1:32:1,32:8192:32" or "64,128" -> sorted unique counts (harness.py:227-253)."""
    values: set[int] = set()
    for part in (p.strip() for p in spec.split(",")):
        if not part:
            continue
        pieces = part.split(":")
        try:
            if len(pieces) == 1:
                values.add(int(pieces[0]))
            elif len(pieces) == 3:
                a, b, st = (int(x) for x in pieces)
                if st < 1 or a < 1 or b < a:
                    raise ValueError(f"bad range {part!r}")
                values.update(range(a, b + 1, st))
            else:
                raise ValueError(f"bad range {part!r}")
        except ValueError as e:
            raise ConfigError(f"cannot parse n_sim spec {spec!r}: {e}") from None
    if not values or min(values) < 1:
        raise ConfigError(f"n_sim spec {spec!r} must produce positive counts")
    return sorted(values)


def bench_sweep(plant, cset, model, template, n_sim_values, backends=("cuda",), reps=20,
                seed=7, modes=_BENCH_MODES, x0=None, v_prev=0.0, r=0.5):
    """Time governor calls over (backend, n_sim) cells on the frozen bench snapshot
    (harness.py:259-355): one untimed warm-up call, then `reps` timed calls of
    robust_rg_parallel on a fresh state; end-to-end draws a fresh scenario set
    inside the clock.  Backends other than the device names yield skipped records
    (this build has no CPU backends)."""
    from .disturbance import derive_seed
    from .governor import BACKENDS, GovernorConfig

    if not n_sim_values or not backends:
        raise ConfigError("n_sim_values and backends must be nonempty")
    if reps < 1:
        raise ConfigError(f"reps must be >= 1, got {reps}")
    for mode in modes:
        if mode not in _BENCH_MODES:
            raise ConfigError(f"unknown timing mode {mode!r}; known: {_BENCH_MODES}")
    x0 = plant.validate_state(np.zeros(plant.state_dim) if x0 is None else x0)
    records = []
    for backend in backends:
        for n_sim in n_sim_values:
            if backend not in BACKENDS:
                records += [TimingRecord(backend, n_sim, template.m_grid, reps, m, None, None,
                                         None, skipped=True) for m in modes]
                continue
            cfg = GovernorConfig(j_star=template.j_star, epsilon=template.epsilon,
                                 n_kappa=template.n_kappa, m_grid=template.m_grid, n_sim=n_sim,
                                 backend=backend, infeasible_policy=template.infeasible_policy,
                                 prefix_mode=template.prefix_mode,
                                 tighten_mode=template.tighten_mode,
                                 device=getattr(template, "device", 0),
                                 keep_matrix=getattr(template, "keep_matrix", True))
            cell_seed = derive_seed(seed, f"bench:{backend}:{n_sim}")
            scen = sample_scenarios(model, n_sim, cfg.j_star + 1, seed=cell_seed,
                                    device=cfg.device)
            for mode in modes:
                robust_rg_parallel(plant, x0, GovernorState(v_prev), r, cset, scen, cfg)
                times = np.empty(reps)
                for i in range(reps):
                    t0 = time.perf_counter()
                    s_ = scen if mode == "kernel-only" else sample_scenarios(
                        model, n_sim, cfg.j_star + 1, seed=cell_seed + i + 1, device=cfg.device)
                    robust_rg_parallel(plant, x0, GovernorState(v_prev), r, cset, s_, cfg)
                    times[i] = (time.perf_counter() - t0) * 1e6
                records.append(TimingRecord(backend, n_sim, cfg.m_grid, reps, mode,
                                            float(times.mean()), float(times.min()),
                                            float(times.max())))
    return records


def _fmt(x) -> str:
    if x is None:
        return ""
    if isinstance(x, bool):
        return str(int(x))
    if isinstance(x, float):
        return repr(x)
    return str(x)


def emit_csv(records, path, kind: str | None = None) -> None:
    """RunRecord -> run CSV, [TimingRecord] -> timing CSV (harness.py:368-414)."""
    if kind is None:
        if isinstance(records, RunRecord):
            kind = "run"
        elif isinstance(records, (list, tuple)) and records and \
                isinstance(records[0], TimingRecord):
            kind = "timing"
        else:
            raise ConfigError("cannot infer CSV schema; pass kind=")
    if kind == "run":
        lines = [RUN_CSV_HEADER] + [",".join(_fmt(v) for v in row) for row in records.rows]
    elif kind == "timing":
        lines = [TIMING_CSV_HEADER] + [",".join([rec.backend, str(rec.n_sim), rec.mode,
                                                 _fmt(rec.mean_us), _fmt(rec.min_us),
                                                 _fmt(rec.max_us), str(rec.reps)])
                                       for rec in records]
    else:
        raise ConfigError(f"unknown CSV kind {kind!r}")
    try:
        with open(path, "w") as f:
            f.write("\n".join(lines) + "\n")
    except OSError as e:
        raise ConfigError(f"cannot write CSV to {path}: {e}") from None
