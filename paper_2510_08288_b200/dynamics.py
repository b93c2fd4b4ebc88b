"""Plants (reference dynamics.py:47-328), host side.

The device kernels specialise on ``kernel_kind == "surrogate-fc"``: the
three-state tanh surrogate of the fuel-cell air path,

    dx1/dt = -x1 + tanh(x2),  dx2/dt = -x2 + v,  dx3/dt = -2 x3 + x1,  y = x1,

discretised with fixed-step RK4.  The prediction rollouts run on the B200
(csrc/rg_cell.cuh); what stays here is what the reference computes with
numpy's tanh: the steady-state map y_ss(v) = tanh(v) (dynamics.py:243-244) and
the true-plant step of the closed loop (dynamics.py:110-130, 228-231).  Both
are kept as numpy so they stay bit-identical with the reference.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import ConfigError, IntegrationOverflowError

__all__ = ["Plant", "SurrogateFuelCellPlant", "LinearOraclePlant", "make_plant",
           "rk4_step", "STATE_ABORT_LIMIT"]

STATE_ABORT_LIMIT = 1e6


class Plant:
    """Discrete-time closed loop under a constant setpoint (dynamics.py:47-87)."""

    state_dim: int = 0
    kernel_kind: str | None = None

    def step(self, x, v):  # pragma: no cover - interface
        raise NotImplementedError

    def output(self, x, v) -> float:  # pragma: no cover - interface
        raise NotImplementedError

    def steady_state_output(self, v) -> float:  # pragma: no cover - interface
        raise NotImplementedError

    def validate_state(self, x) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.state_dim,):
            raise ConfigError(f"state must have shape ({self.state_dim},), got {x.shape}")
        if not all(map(math.isfinite, x.tolist())):
            raise ConfigError("state entries must be finite")
        return x


def _surrogate_rhs(x: np.ndarray, v: float) -> np.ndarray:
    # dynamics.py:228-231, numpy tanh on a float64 scalar
    return np.array([-x[0] + np.tanh(x[1]), -x[1] + v, -2.0 * x[2] + x[0]], dtype=np.float64)


def rk4_step(plant, x: np.ndarray, v: float) -> np.ndarray:
    """One RK4 step x + (h/6)(k1 + 2k2 + 2k3 + k4) of the surrogate, with the
    reference's overflow check (dynamics.py:110-130)."""
    h = plant.step_size
    k1 = _surrogate_rhs(x, v)
    k2 = _surrogate_rhs(x + 0.5 * h * k1, v)
    k3 = _surrogate_rhs(x + 0.5 * h * k2, v)
    k4 = _surrogate_rhs(x + h * k3, v)
    nxt = x + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    bad = ~np.isfinite(nxt) | (np.abs(nxt) > STATE_ABORT_LIMIT)
    if bad.any():
        i = int(np.argmax(bad))
        raise IntegrationOverflowError(f"integration overflow in state {i} (value {nxt[i]!r})",
                                       state_index=i)
    return nxt


def _surrogate_rk4(h: float, x: np.ndarray, v: float) -> np.ndarray:
    """rk4_step for the surrogate in Python floats: the reference's elementwise numpy
    operations one element at a time, same operands, same order, same roundings (CPython
    floats are IEEE doubles without contraction).  dx2/dt = -x2 + v does not involve the
    other states, so the four stage values of x2 -- the four tanh arguments -- come first
    and go through ONE numpy tanh call (numpy's vector tanh equals its scalar tanh bit for
    bit, tests/test_harness_batch.py).  ~5x cheaper than the 3-element array form, once per
    closed-loop step (dynamics.py:110-130, 228-231)."""
    hh = 0.5 * h
    x0, x1, x2 = float(x[0]), float(x[1]), float(x[2])
    k11 = -x1 + v
    b1 = x1 + hh * k11
    k21 = -b1 + v
    c1 = x1 + hh * k21
    k31 = -c1 + v
    d1 = x1 + h * k31
    k41 = -d1 + v
    t1, t2, t3, t4 = np.tanh(np.array([x1, b1, c1, d1])).tolist()
    k10 = -x0 + t1
    k12 = -2.0 * x2 + x0
    a0, a2 = x0 + hh * k10, x2 + hh * k12
    k20 = -a0 + t2
    k22 = -2.0 * a2 + a0
    b0, b2 = x0 + hh * k20, x2 + hh * k22
    k30 = -b0 + t3
    k32 = -2.0 * b2 + b0
    c0, c2 = x0 + h * k30, x2 + h * k32
    k40 = -c0 + t4
    k42 = -2.0 * c2 + c0
    c = h / 6.0
    nxt = np.array([x0 + c * (((k10 + 2.0 * k20) + 2.0 * k30) + k40),
                    x1 + c * (((k11 + 2.0 * k21) + 2.0 * k31) + k41),
                    x2 + c * (((k12 + 2.0 * k22) + 2.0 * k32) + k42)])
    bad = ~np.isfinite(nxt) | (np.abs(nxt) > STATE_ABORT_LIMIT)
    if bad.any():
        i = int(np.argmax(bad))
        raise IntegrationOverflowError(f"integration overflow in state {i} (value {nxt[i]!r})",
                                       state_index=i)
    return nxt


class SurrogateFuelCellPlant(Plant):
    """RK4-discretised surrogate benchmark plant (dynamics.py:209-263)."""

    kernel_kind = "surrogate-fc"
    state_dim = 3

    def __init__(self, step_size: float = 0.01):
        if not step_size > 0:
            raise ConfigError(f"step_size must be positive, got {step_size}")
        self.step_size = float(step_size)

    def step(self, x, v):
        return _surrogate_rk4(self.step_size, np.asarray(x, dtype=np.float64), float(v))

    def output(self, x, v) -> float:
        return float(x[0])

    def steady_state_output(self, v) -> float:
        return float(np.tanh(v))


class LinearOraclePlant(Plant):
    """x+ = A x + B v, y = C x + D v (dynamics.py:162-206).

    Host-only here: the device kernels cover the surrogate plant, which is the
    hot path; passing this plant to a device governor raises
    BackendUnavailableError exactly as the reference's GPU backend does
    (backend_gpu.py:66-71).
    """

    kernel_kind = "linear"

    def __init__(self, A, B, C, D: float = 0.0):
        A = np.atleast_2d(np.asarray(A, dtype=np.float64))
        B = np.asarray(B, dtype=np.float64).reshape(-1)
        C = np.asarray(C, dtype=np.float64).reshape(-1)
        n = A.shape[0]
        if A.shape != (n, n):
            raise ConfigError(f"A must be square, got {A.shape}")
        if B.shape != (n,) or C.shape != (n,):
            raise ConfigError("B and C must be length-n vectors")
        if n and float(np.max(np.abs(np.linalg.eigvals(A)))) >= 1.0:
            raise ConfigError("A must have spectral radius < 1")
        self.A, self.B, self.C, self.D = A, B, C, float(D)
        self.state_dim = n
        self.dc_gain = float(C @ np.linalg.solve(np.eye(n) - A, B) + self.D)

    def step(self, x, v):
        return self.A @ x + self.B * v

    def output(self, x, v) -> float:
        return float(self.C @ x + self.D * v)

    def steady_state_output(self, v) -> float:
        return self.dc_gain * v


def make_plant(kind: str, **kwargs) -> Plant:
    """Plant by identifier (dynamics.py:317-328)."""
    if kind == "surrogate-fc":
        return SurrogateFuelCellPlant(step_size=kwargs.get("step_size", 0.01))
    if kind == "linear-oracle":
        missing = [k for k in ("A", "B", "C") if k not in kwargs]
        if missing:
            raise ConfigError(f"linear-oracle plant requires matrices {missing}")
        return LinearOraclePlant(kwargs["A"], kwargs["B"], kwargs["C"], kwargs.get("D", 0.0))
    raise ConfigError(f"unknown plant kind {kind!r}; known: ['linear-oracle', 'surrogate-fc']")
