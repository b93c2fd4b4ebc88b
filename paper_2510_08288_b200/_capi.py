"""ctypes binding of the C ABI (include/refgov_b200.h).

The library is built in-tree (``python -m paper_2510_08288_b200.build`` or
``__graft_entry__.build()``) as ``_lib/librefgov_b200.so``.  There is no
fallback: if the library or a CUDA device is missing, every device entry point
raises BackendUnavailableError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import BackendUnavailableError, ConfigError, RefgovError

LIB_PATH = Path(os.environ.get("RG_LIB_PATH") or
                Path(__file__).resolve().parent / "_lib" / "librefgov_b200.so")

RG_OK, RG_E_NODEVICE, RG_E_UNSUPPORTED, RG_E_ARGS, RG_E_CUDA = 0, -1, -2, -3, -4
RG_TANH_AUTO, RG_TANH_FMA, RG_TANH_GENERIC = 0, 1, 2
RG_DEVICE_PTRS, RG_ASYNC, RG_ABANDON, RG_NO_TIMING = 0x1, 0x2, 0x4, 0x8
RG_TANH_LOCKSTEP, RG_FUSED_RNG, RG_STAGE_RNG = 0x10, 0x20, 0x40
RG_JOINT_ITER = 0x80
RG_XCHG = 0x100
XCHG_HANDLE_BYTES = 64  # sizeof(cudaIpcMemHandle_t)
_RNG_FLAGS = {None: 0, "fused": RG_FUSED_RNG, "staged": RG_STAGE_RNG}

_i32, _i64, _u64, _d, _vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, \
    ctypes.c_void_p


class Problem(ctypes.Structure):
    _fields_ = [("step_size", _d), ("y_lower", _d), ("y_upper", _d), ("ss_v_lower", _d),
                ("ss_v_upper", _d), ("j_star", _i32), ("_pad", _i32)]


class Scenarios(ctypes.Structure):
    _fields_ = [("seed", _u64), ("k0", _i64), ("n_sim", _i64), ("lo", _d * 4), ("span", _d * 4)]


class LinearPlant(ctypes.Structure):
    _fields_ = [("n", _i32), ("_pad", _i32), ("A", _d * 16), ("B", _d * 4), ("C", _d * 4),
                ("D", _d), ("dc_gain", _d), ("ss_lower", _d), ("ss_upper", _d)]


def make_linear(plant, ss_lower: float, ss_upper: float) -> "LinearPlant":
    """rg_linear_plant for a LinearOraclePlant (n <= 4 states)."""
    n = int(plant.state_dim)
    if not 1 <= n <= 4:
        raise BackendUnavailableError(f"the device linear kernels support 1..4 states, got {n}")
    A = np.zeros(16)
    A[: n * n] = np.asarray(plant.A, dtype=np.float64).reshape(-1)
    B = np.zeros(4)
    B[:n] = plant.B
    C = np.zeros(4)
    C[:n] = plant.C
    d16, d4 = _d * 16, _d * 4
    return LinearPlant(n, 0, d16(*A), d4(*B), d4(*C), float(plant.D), float(plant.dc_gain),
                       float(ss_lower), float(ss_upper))


class GridResult(ctypes.Structure):
    _fields_ = [("row", _i32), ("n_active", _i32), ("ss_pruned_rows", _i32),
                ("dedup_rows", _i32), ("sims_run", _i64), ("early_terms", _i64),
                ("overflows", _i64), ("abandoned", _i64), ("kernel_ms", ctypes.c_float),
                ("reduce_us", ctypes.c_float)]


class LoopResult(ctypes.Structure):
    _fields_ = [("steps_done", _i32), ("abort_kind", _i32), ("abort_step", _i32),
                ("abort_index", _i32), ("abort_value", _d)]


RG_LOOP_OVERFLOW, RG_LOOP_LEFT_BOX, RG_LOOP_INFEASIBLE = 1, 2, 3


class BisectResult(ctypes.Structure):
    _fields_ = [("kappa", _d), ("found", _i32), ("_pad", _i32), ("cells", _i64),
                ("early", _i64), ("kernel_ms", ctypes.c_float), ("_pad2", _i32)]


_RANGE4: dict = {}


def _range4(lo, span):
    """The padded double[4] lo/span pair, cached by value (bytes of the float64 arrays)."""
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    span = np.ascontiguousarray(span, dtype=np.float64)
    key = (lo.tobytes(), span.tobytes())
    r = _RANGE4.get(key)
    if r is None:
        d4 = _d * 4
        a = lo.tolist() + [0.0] * (4 - lo.size)
        b = span.tolist() + [0.0] * (4 - span.size)
        if len(_RANGE4) > 256:
            _RANGE4.clear()
            _SCEN_TEMPLATE.clear()
        r = _RANGE4[key] = (d4(*a[:4]), d4(*b[:4]))
    return r


_SCEN_TEMPLATE: dict = {}


def make_scenarios(seed: int, k0: int, n_sim: int, lo, span) -> "Scenarios":
    """rg_scenarios for the counter-RNG stream ``seed`` (masked to 64 bits)."""
    lo4, span4 = _range4(lo, span)
    t = _SCEN_TEMPLATE.get((id(lo4), id(span4)))
    if t is None:  # one template per cached range pair; copying it is cheaper than a build
        t = _SCEN_TEMPLATE[(id(lo4), id(span4))] = (Scenarios(0, 0, 0, lo4, span4), lo4, span4)
    s = Scenarios.from_buffer_copy(t[0])
    s.seed = int(seed) & (2**64 - 1)
    s.k0 = int(k0)
    s.n_sim = int(n_sim)
    return s


# name -> (restype, argtypes); the exact export list of include/refgov_b200.h
SIGNATURES = {
    "rg_abi_version": (_i32, []),
    "rg_last_error": (ctypes.c_char_p, []),
    "rg_device_count": (_i32, [ctypes.POINTER(_i32)]),
    "rg_create": (_i32, [_i32, _i32, ctypes.POINTER(_vp)]),
    "rg_destroy": (_i32, [_vp]),
    "rg_get_tanh_variant": (_i32, [_vp, ctypes.POINTER(_i32)]),
    "rg_set_option": (_i32, [_vp, ctypes.c_char_p, _i64]),
    "rg_get_option": (_i32, [_vp, ctypes.c_char_p, ctypes.POINTER(_i64)]),
    "rg_get_stream": (_i32, [_vp, ctypes.POINTER(_vp)]),
    "rg_closed_loop": (_i32, [_vp, ctypes.POINTER(Problem), _i32, _i32, _i32, _vp, _d, _i32,
                              _vp, _vp, _u64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                              _vp, _vp, ctypes.POINTER(LoopResult)]),
    "rg_closed_loop_bisection": (_i32, [_vp, ctypes.POINTER(Problem), _i32, _vp, _d, _i32, _vp,
                                        _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                        ctypes.POINTER(LoopResult)]),
    "rg_np_tanh": (_i32, [_vp, _vp, _i64]),
    "rg_plant_step": (_i32, [_d, _vp, _d, _vp]),
    "rg_synchronize": (_i32, [_vp]),
    "rg_tanh": (_i32, [_vp, _vp, _vp, _i64, _i32]),
    "rg_sample_scenarios": (_i32, [_vp, _u64, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _i32]),
    "rg_fill": (_i32, [_vp, ctypes.POINTER(Problem), _vp, _vp, _i32, _vp, _i32, _vp, _i64,
                       _i64, ctypes.POINTER(Scenarios), _vp, _vp, _i32]),
    "rg_grid_step": (_i32, [_vp, ctypes.POINTER(Problem), _vp, _d, _d, _i32, _i32, _vp, _i64,
                            _i64, ctypes.POINTER(Scenarios), _vp, _vp,
                            ctypes.POINTER(GridResult), _i32]),
    "rg_grid_fetch": (_i32, [_vp, _vp, _i32, ctypes.POINTER(GridResult)]),
    "rg_bisect": (_i32, [_vp, ctypes.POINTER(Problem), _vp, _d, _d, _i32, _vp, _i64, _i64,
                         ctypes.POINTER(Scenarios), _vp, _vp, _vp, _vp, _vp, _vp,
                         ctypes.POINTER(BisectResult), _i32]),
    "rg_grid_step_batch": (_i32, [_vp, ctypes.POINTER(Problem), _i32, _vp, _vp, _vp, _vp, _i64,
                                  _i64, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _i32]),
    "rg_fill_linear": (_i32, [_vp, ctypes.POINTER(LinearPlant), ctypes.POINTER(Problem), _vp,
                              _vp, _i32, _vp, _i32, _vp, _i64, _i64, ctypes.POINTER(Scenarios),
                              _vp, _vp, _i32]),
    "rg_bisect_linear": (_i32, [_vp, ctypes.POINTER(LinearPlant), ctypes.POINTER(Problem), _vp,
                                _d, _d, _i32, _vp, _i64, _i64, ctypes.POINTER(Scenarios), _vp,
                                _vp, _vp, _vp, ctypes.POINTER(BisectResult), _i32]),
    "rg_bisect_joint": (_i32, [_vp, ctypes.POINTER(Problem), _vp, _d, _d, _i32, _vp, _i64, _i64,
                               ctypes.POINTER(Scenarios), ctypes.POINTER(BisectResult), _i32]),
    "rg_joint_begin": (_i32, [_vp, ctypes.POINTER(Problem), _vp, _d, _d, _i32, _vp, _i64, _i64,
                              ctypes.POINTER(Scenarios), _i32]),
    "rg_joint_iter": (_i32, [_vp, _i32, _i32]),
    "rg_joint_flag": (_i32, [_vp, ctypes.POINTER(_vp)]),
    "rg_joint_decide": (_i32, [_vp, _i32]),
    "rg_joint_end": (_i32, [_vp, ctypes.POINTER(BisectResult)]),
    "rg_xchg_init": (_i32, [_vp, _i32, _i32, _vp]),
    "rg_xchg_connect": (_i32, [_vp, _vp]),
    "rg_xchg_close": (_i32, [_vp]),
    "rg_bisect_joint_sharded": (_i32, [_vp, ctypes.POINTER(Problem), _vp, _d, _d, _i32, _vp, _i64,
                                       _i64, ctypes.POINTER(Scenarios), _i64,
                                       ctypes.POINTER(BisectResult), _i32]),
    "rg_fp64_peak": (_i32, [_vp, ctypes.POINTER(_d)]),
}

_lib = None
_lock = threading.RLock()
_contexts: dict = {}


def load_library():
    """Load the in-tree CUDA library; BackendUnavailableError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise BackendUnavailableError(
                f"CUDA library {LIB_PATH} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.rg_abi_version() != 1:
            raise BackendUnavailableError("CUDA library ABI version mismatch; rebuild it")
        _lib = lib
        return lib


def check(code: int) -> None:
    if code == RG_OK:
        return
    msg = (_lib.rg_last_error() or b"").decode(errors="replace")
    if code in (RG_E_NODEVICE, RG_E_UNSUPPORTED):
        raise BackendUnavailableError(msg)
    if code == RG_E_ARGS:
        raise ConfigError(msg)
    raise RefgovError(f"CUDA failure: {msg}")


def _p(a: np.ndarray | None):
    # the integer address: ctypes passes it for c_void_p arguments, and it is
    # several times cheaper to produce than a.ctypes.data_as(c_void_p)
    return None if a is None else a.ctypes.data


def np_tanh(x) -> np.ndarray:
    """numpy's float64 tanh restated in the library (rg_np_tanh, host code, no device)."""
    lib = load_library()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    check(lib.rg_np_tanh(_p(x), _p(y), x.size))
    return y


def plant_step(step_size: float, x, v: float) -> np.ndarray:
    """The surrogate true plant's RK4 step in the library (rg_plant_step, host code)."""
    lib = load_library()
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(3)
    check(lib.rg_plant_step(float(step_size), _p(x), float(v), _p(out)))
    return out


def device_count() -> int:
    lib = load_library()
    n = _i32(0)
    rc = lib.rg_device_count(ctypes.byref(n))
    return int(n.value) if rc == RG_OK else 0


def _locked(fn):
    """Hold the context's lock for the whole call: an rg_ctx serves one call at a
    time (its scratch buffers, pinned result block and publication token are
    shared), and ctypes releases the GIL while the C function runs."""
    import functools

    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        with self.lock:
            return fn(self, *args, **kwargs)

    return wrapper


class Context:
    """One CUDA context per device: stream, scratch buffers, result staging.

    Thread-safe: every entry point holds ``lock`` (re-entrant), so concurrent
    governor calls on one device -- the reference service runs /govern/step in a
    thread pool -- are serialised instead of racing on the shared scratch.  A
    caller issuing a sequence of calls that must not interleave (the sharded
    joint search) holds ``lock`` around the sequence.
    """

    def __init__(self, device: int = 0, tanh_variant: int = RG_TANH_AUTO):
        self.lock = threading.RLock()
        self.lib = load_library()
        h = _vp()
        check(self.lib.rg_create(int(device), int(tanh_variant), ctypes.byref(h)))
        self.handle = h
        self.device = int(device)
        v = _i32()
        check(self.lib.rg_get_tanh_variant(self.handle, ctypes.byref(v)))
        self.tanh_variant = int(v.value)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.rg_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream_ptr(self) -> int:
        s = _vp()
        check(self.lib.rg_get_stream(self.handle, ctypes.byref(s)))
        return int(s.value or 0)

    @_locked
    def synchronize(self):
        check(self.lib.rg_synchronize(self.handle))

    @_locked
    def set_option(self, name: str, value: int) -> None:
        """rg_set_option: a tuning knob of this context (no result bit depends on it)."""
        check(self.lib.rg_set_option(self.handle, name.encode(), int(value)))

    @_locked
    def get_option(self, name: str) -> int:
        """rg_get_option: a tuning knob, or "last_grid_kernel" (0 k_grid, 1 k_grid_ts)."""
        v = _i64(0)
        check(self.lib.rg_get_option(self.handle, name.encode(), ctypes.byref(v)))
        return int(v.value)

    # -- entry points ---------------------------------------------------
    @_locked
    def tanh(self, x: np.ndarray, lockstep: bool = False) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        check(self.lib.rg_tanh(self.handle, _p(x), _p(y), x.size,
                               RG_TANH_LOCKSTEP if lockstep else 0))
        return y

    @_locked
    def sample(self, seed: int, k0: int, n_sim: int, horizon: int, lo, span) -> np.ndarray:
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        span = np.ascontiguousarray(span, dtype=np.float64)
        out = np.empty((n_sim, horizon, lo.size), dtype=np.float64)
        check(self.lib.rg_sample_scenarios(self.handle, seed & (2**64 - 1), k0, n_sim, horizon,
                                           lo.size, _p(lo), _p(span), _p(out), 0))
        return out

    @_locked
    def fill(self, prob: Problem, x0, v_rows, rows, dist, n_sim, scen: Scenarios | None,
             S: np.ndarray, steps: np.ndarray, rng_mode: str | None = None) -> None:
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        v_rows = np.ascontiguousarray(v_rows, dtype=np.float64)
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        horizon = 0
        if dist is not None:
            dist = np.ascontiguousarray(dist, dtype=np.float64)
            horizon = dist.shape[1]
        check(self.lib.rg_fill(self.handle, ctypes.byref(prob), _p(x0), _p(v_rows), v_rows.size,
                               _p(rows), rows.size, _p(dist), int(n_sim), int(horizon),
                               ctypes.byref(scen) if scen is not None else None, _p(S),
                               _p(steps), _RNG_FLAGS[rng_mode]))

    @_locked
    def grid_step(self, prob: Problem, x0, v_prev, r, m_grid, prefix_mode, dist, n_sim,
                  scen: Scenarios | None, want_pbits: bool, abandon: bool = False,
                  rng_mode: str | None = None, timing: bool = True, want_viol: bool = True,
                  xchg: bool = False):
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        horizon = 0
        if dist is not None:
            dist = np.ascontiguousarray(dist, dtype=np.float64)
            horizon = dist.shape[1]
        viol = np.empty(m_grid, dtype=np.uint32) if want_viol else None
        pbits = np.empty((m_grid, (n_sim + 31) // 32), dtype=np.uint32) if want_pbits else None
        res = GridResult()
        flags = (RG_ABANDON if abandon else 0) | _RNG_FLAGS[rng_mode] | \
            (0 if timing else RG_NO_TIMING) | (RG_XCHG if xchg else 0)
        check(self.lib.rg_grid_step(self.handle, ctypes.byref(prob), _p(x0), float(v_prev),
                                    float(r), int(m_grid), int(bool(prefix_mode)), _p(dist),
                                    int(n_sim), int(horizon),
                                    ctypes.byref(scen) if scen is not None else None, _p(viol),
                                    _p(pbits), ctypes.byref(res), flags))
        return res, viol, pbits

    @_locked
    def grid_step_to_device(self, prob: Problem, x0, v_prev, r, m_grid, prefix_mode, n_sim,
                            scen: Scenarios, viol_dev: int, abandon: bool = True) -> None:
        """Enqueue a grid step on the library's stream; the per-row violation
        counts (uint32, 0xffffffff = gated out) land at the device address
        `viol_dev`.  No host synchronisation (RG_ASYNC | RG_DEVICE_PTRS)."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        res = GridResult()
        check(self.lib.rg_grid_step(self.handle, ctypes.byref(prob), _p(x0), float(v_prev),
                                    float(r), int(m_grid), int(bool(prefix_mode)), None,
                                    int(n_sim), 0, ctypes.byref(scen), ctypes.c_void_p(viol_dev),
                                    None, ctypes.byref(res),
                                    RG_ASYNC | RG_DEVICE_PTRS | RG_NO_TIMING
                                    | (RG_ABANDON if abandon else 0)))

    @_locked
    def bisect(self, prob: Problem, x0, v_prev, r, n_kappa, dist, n_sim,
               scen: Scenarios | None, per_scenario: bool = False, paths: bool = False,
               rng_mode: str | None = None):
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        horizon = 0
        if dist is not None:
            dist = np.ascontiguousarray(dist, dtype=np.float64)
            horizon = dist.shape[1]
        kap = fnd = cel = erl = pk = po = None
        if per_scenario:
            kap = np.empty(n_sim, dtype=np.float64)
            fnd = np.empty(n_sim, dtype=np.int32)
            cel = np.empty(n_sim, dtype=np.int32)
            erl = np.empty(n_sim, dtype=np.int32)
        if paths:
            pk = np.empty((n_sim, n_kappa + 1), dtype=np.float64)
            po = np.empty((n_sim, n_kappa + 1), dtype=np.uint8)
        res = BisectResult()
        check(self.lib.rg_bisect(self.handle, ctypes.byref(prob), _p(x0), float(v_prev), float(r),
                                 int(n_kappa), _p(dist), int(n_sim), int(horizon),
                                 ctypes.byref(scen) if scen is not None else None, _p(kap),
                                 _p(fnd), _p(cel), _p(erl), _p(pk), _p(po), ctypes.byref(res),
                                 _RNG_FLAGS[rng_mode]))
        per = (kap, fnd, cel, erl) if per_scenario else None
        return res, per, ((pk, po) if paths else None)

    @_locked
    def bisect_joint(self, prob: Problem, x0, v_prev, r, n_kappa, dist, n_sim,
                     scen: Scenarios | None, rng_mode: str | None = None,
                     per_iteration: bool = False) -> "BisectResult":
        """Joint bisection on this device (rg_bisect_joint): one persistent kernel, or
        one kernel per iteration with `per_iteration`."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        horizon = 0
        if dist is not None:
            dist = np.ascontiguousarray(dist, dtype=np.float64)
            horizon = dist.shape[1]
        res = BisectResult()
        check(self.lib.rg_bisect_joint(self.handle, ctypes.byref(prob), _p(x0), float(v_prev),
                                       float(r), int(n_kappa), _p(dist), int(n_sim),
                                       int(horizon),
                                       ctypes.byref(scen) if scen is not None else None,
                                       ctypes.byref(res), _RNG_FLAGS[rng_mode]
                                       | (RG_JOINT_ITER if per_iteration else 0)))
        return res

    @_locked
    def joint_begin(self, prob: Problem, x0, v_prev, r, n_kappa, dist, n_sim,
                    scen: Scenarios | None) -> None:
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        horizon = 0
        if dist is not None:
            dist = np.ascontiguousarray(dist, dtype=np.float64)
            horizon = dist.shape[1]
        check(self.lib.rg_joint_begin(self.handle, ctypes.byref(prob), _p(x0), float(v_prev),
                                      float(r), int(n_kappa), _p(dist), int(n_sim),
                                      int(horizon),
                                      ctypes.byref(scen) if scen is not None else None, 0))

    @_locked
    def joint_iter(self, it: int, fold: bool) -> None:
        check(self.lib.rg_joint_iter(self.handle, int(it), int(bool(fold))))

    @_locked
    def joint_flag_ptr(self) -> int:
        p = _vp()
        check(self.lib.rg_joint_flag(self.handle, ctypes.byref(p)))
        return int(p.value)

    @_locked
    def joint_decide(self, it: int) -> None:
        check(self.lib.rg_joint_decide(self.handle, int(it)))

    @_locked
    def joint_end(self) -> "BisectResult":
        res = BisectResult()
        check(self.lib.rg_joint_end(self.handle, ctypes.byref(res)))
        return res

    @_locked
    def grid_step_batch(self, prob: Problem, x0, v_prev, r, seeds, k0, n_sim, lo, span,
                        m_grid, prefix_mode=False, abandon=True, want_viol=False, fused=False,
                        staged=False):
        """Batched robust grid step; returns (row, kappa, v, early[, viol]).  The library
        stages each episode's scenario block when more than two rows per episode are live
        and fuses the RNG into the rollouts otherwise; `fused` / `staged` force one."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64).reshape(-1, 3)
        E = x0.shape[0]
        v_prev = np.ascontiguousarray(v_prev, dtype=np.float64).reshape(E)
        r = np.ascontiguousarray(r, dtype=np.float64).reshape(E)
        seeds = np.asarray([int(s_) & (2**64 - 1) for s_ in seeds], dtype=np.uint64)
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        span = np.ascontiguousarray(span, dtype=np.float64)
        row = np.empty(E, np.int32)
        kap = np.empty(E, np.float64)
        v = np.empty(E, np.float64)
        early = np.empty(E, np.int64)
        viol = np.empty((E, m_grid), np.uint32) if want_viol else None
        check(self.lib.rg_grid_step_batch(self.handle, ctypes.byref(prob), E, _p(x0), _p(v_prev),
                                          _p(r), _p(seeds), int(k0), int(n_sim), _p(lo),
                                          _p(span), int(m_grid), int(bool(prefix_mode)),
                                          _p(row), _p(kap), _p(v), _p(early), _p(viol),
                                          (RG_ABANDON if abandon else 0)
                                          | (RG_FUSED_RNG if fused else 0)
                                          | (RG_STAGE_RNG if staged else 0)))
        return (row, kap, v, early, viol) if want_viol else (row, kap, v, early)

    @_locked
    def fill_linear(self, lin: LinearPlant, prob: Problem, x0, v_rows, rows, dist, n_sim,
                    scen: Scenarios | None, S: np.ndarray, steps: np.ndarray) -> None:
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        v_rows = np.ascontiguousarray(v_rows, dtype=np.float64)
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        horizon = 0
        if dist is not None:
            dist = np.ascontiguousarray(dist, dtype=np.float64)
            horizon = dist.shape[1]
        check(self.lib.rg_fill_linear(self.handle, ctypes.byref(lin), ctypes.byref(prob), _p(x0),
                                      _p(v_rows), v_rows.size, _p(rows), rows.size, _p(dist),
                                      int(n_sim), int(horizon),
                                      ctypes.byref(scen) if scen is not None else None, _p(S),
                                      _p(steps), 0))

    @_locked
    def bisect_linear(self, lin: LinearPlant, prob: Problem, x0, v_prev, r, n_kappa, dist,
                      n_sim, scen: Scenarios | None, per_scenario: bool = False):
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        horizon = 0
        if dist is not None:
            dist = np.ascontiguousarray(dist, dtype=np.float64)
            horizon = dist.shape[1]
        kap = fnd = cel = erl = None
        if per_scenario:
            kap = np.empty(n_sim, dtype=np.float64)
            fnd = np.empty(n_sim, dtype=np.int32)
            cel = np.empty(n_sim, dtype=np.int32)
            erl = np.empty(n_sim, dtype=np.int32)
        res = BisectResult()
        check(self.lib.rg_bisect_linear(self.handle, ctypes.byref(lin), ctypes.byref(prob),
                                        _p(x0), float(v_prev), float(r), int(n_kappa), _p(dist),
                                        int(n_sim), int(horizon),
                                        ctypes.byref(scen) if scen is not None else None,
                                        _p(kap), _p(fnd), _p(cel), _p(erl), ctypes.byref(res),
                                        0))
        return res, ((kap, fnd, cel, erl) if per_scenario else None)

    @_locked
    def xchg_init(self, rank: int, world: int) -> bytes:
        """rg_xchg_init: allocate this rank's exchange window; its CUDA IPC handle."""
        h = ctypes.create_string_buffer(XCHG_HANDLE_BYTES)
        check(self.lib.rg_xchg_init(self.handle, int(rank), int(world), h))
        return h.raw

    @_locked
    def xchg_connect(self, handles: bytes) -> None:
        """rg_xchg_connect: map every rank's window (handles rank-major, 64 bytes each)."""
        buf = ctypes.create_string_buffer(bytes(handles), len(handles))
        check(self.lib.rg_xchg_connect(self.handle, buf))

    @_locked
    def bisect_joint_sharded(self, prob: Problem, x0, v_prev, r, n_kappa, dist, n_sim,
                             scen: Scenarios | None, n_sim_max: int) -> "BisectResult":
        """rg_bisect_joint_sharded: this rank's shard of a joint search, the per-round
        exchange fused into the persistent kernel (needs xchg_connect)."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        horizon = 0
        if dist is not None:
            dist = np.ascontiguousarray(dist, dtype=np.float64)
            horizon = dist.shape[1]
        res = BisectResult()
        check(self.lib.rg_bisect_joint_sharded(self.handle, ctypes.byref(prob), _p(x0),
                                               float(v_prev), float(r), int(n_kappa), _p(dist),
                                               int(n_sim), int(horizon),
                                               ctypes.byref(scen) if scen is not None else None,
                                               int(n_sim_max), ctypes.byref(res), 0))
        return res

    @_locked
    def xchg_close(self) -> None:
        check(self.lib.rg_xchg_close(self.handle))

    @_locked
    @_locked
    def closed_loop(self, prob: Problem, m_grid: int, prefix_mode: bool, infeasible_error: bool,
                    x0, v0: float, r, d_true, scen_seed: int, n_sim: int, lo, span):
        """rg_closed_loop: the governed loop in native code.  Returns (LoopResult, dict of
        per-step arrays over the steps done, final state)."""
        r = np.ascontiguousarray(r, dtype=np.float64)
        steps = r.size
        d_true = np.ascontiguousarray(d_true, dtype=np.float64).reshape(steps, 3)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        lo3 = np.ascontiguousarray(np.asarray(lo, dtype=np.float64)[:3])
        span3 = np.ascontiguousarray(np.asarray(span, dtype=np.float64)[:3])
        out = {"v": np.empty(steps), "kappa": np.empty(steps), "y": np.empty(steps),
               "feasible": np.empty(steps, dtype=np.uint8),
               "sims_run": np.empty(steps, dtype=np.int64),
               "early_terms": np.empty(steps, dtype=np.int64),
               "wall_us": np.empty(steps, dtype=np.int32)}
        xf = np.empty(3)
        res = LoopResult()
        check(self.lib.rg_closed_loop(
            self.handle, prob, int(m_grid), 1 if prefix_mode else 0, 1 if infeasible_error else 0,
            _p(x0), float(v0), steps, _p(r), _p(d_true), int(scen_seed) & (2**64 - 1), int(n_sim),
            _p(lo3), _p(span3), _p(out["v"]), _p(out["kappa"]), _p(out["y"]),
            _p(out["feasible"]), _p(out["sims_run"]), _p(out["early_terms"]), _p(out["wall_us"]),
            _p(xf), ctypes.byref(res)))
        n = res.steps_done
        return res, {k: a[:n] for k, a in out.items()}, xf

    @_locked
    def closed_loop_bisection(self, prob: Problem, n_kappa: int, x0, v0: float, r, d_true):
        """rg_closed_loop_bisection: the nominal bisection governor's loop (C1) on the device.
        Returns (LoopResult, dict of per-step arrays over the steps done, final state)."""
        r = np.ascontiguousarray(r, dtype=np.float64)
        steps = r.size
        d_true = np.ascontiguousarray(d_true, dtype=np.float64).reshape(steps, 3)
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        out = {"kappa": np.empty(steps), "v": np.empty(steps), "y": np.empty(steps),
               "found": np.empty(steps, dtype=np.uint8),
               "cells": np.empty(steps, dtype=np.int64),
               "early": np.empty(steps, dtype=np.int64),
               "wall_us": np.empty(steps, dtype=np.int32)}
        xf = np.empty(3)
        res = LoopResult()
        check(self.lib.rg_closed_loop_bisection(
            self.handle, prob, int(n_kappa), _p(x0), float(v0), steps, _p(r), _p(d_true),
            _p(out["kappa"]), _p(out["v"]), _p(out["y"]), _p(out["found"]), _p(out["cells"]),
            _p(out["early"]), _p(out["wall_us"]), _p(xf), ctypes.byref(res)))
        n = res.steps_done
        return res, {k: a[:n] for k, a in out.items()}, xf

    def fp64_peak(self) -> float:
        f = _d()
        check(self.lib.rg_fp64_peak(self.handle, ctypes.byref(f)))
        return float(f.value)


def context(device: int = 0) -> Context:
    """The process-wide context of ``device`` (created on first use)."""
    ctx = _contexts.get(device)
    if ctx is None:
        with _lock:
            ctx = _contexts.get(device)
            if ctx is None:
                ctx = Context(device)
                _contexts[device] = ctx
    return ctx
