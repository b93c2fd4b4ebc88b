"""Disturbance scenarios (reference disturbance.py:35-210), generated on the device.

The reference draws scenario tensors on the host with a counter-based
splitmix64 chain (about 51 ms per 1k scenarios at j*=256, 73% of a 10k
closed-loop step -- SURVEY.md §0 fact 5).  Here ``sample_scenarios`` returns a
*generated* ScenarioSet: it records (seed, model, n_sim, horizon) and the
governor kernels regenerate every entry in registers from the same counter
stream, so the tensor never exists in memory.  ``.data`` materialises the
identical (n_sim, horizon, n) float64 array on demand (device kernel + copy),
bit for bit what the reference's ``sample_scenarios`` returns.

Dense ScenarioSets (caller-provided arrays, e.g. from the reference itself)
are staged to the device in SoA layout instead.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

__all__ = ["splitmix64", "counter_uniform", "derive_seed", "DisturbanceModel", "ScenarioSet",
           "sample_scenarios", "zero_scenarios"]

_M64 = (1 << 64) - 1


def splitmix64(z: int) -> int:
    """The splitmix64 finalizer on a Python int (disturbance.py:41-46)."""
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def counter_uniform(seed: int, k: int, j: int, i: int) -> float:
    """u in [0, 1) at (seed, k, j, i) (disturbance.py:49-61)."""
    h = splitmix64(seed & _M64)
    for c in (k, j, i):
        h = splitmix64((h ^ c) & _M64)
    return (h >> 11) * 2.0**-53


def derive_seed(master: int, label: str) -> int:
    """Stream seed from a master seed and a label (disturbance.py:64-69)."""
    h = splitmix64(master & _M64)
    for b in label.encode("utf-8"):
        h = splitmix64((h ^ b) & _M64)
    return h


@dataclass(frozen=True)
class DisturbanceModel:
    """One uniform (lo, hi) range per state (disturbance.py:98-132)."""

    ranges: tuple
    kind: str = "uniform"

    def __post_init__(self):
        try:
            rr = tuple((float(a), float(b)) for a, b in self.ranges)
        except (TypeError, ValueError) as e:
            raise ConfigError(f"ranges must be (lo, hi) pairs: {e}") from None
        if not rr:
            raise ConfigError("ranges must have at least one (lo, hi) pair")
        for i, (a, b) in enumerate(rr):
            if not (np.isfinite(a) and np.isfinite(b)):
                raise ConfigError(f"range {i} must be finite, got ({a}, {b})")
            if a > b:
                raise ConfigError(f"range {i} has lo > hi: ({a}, {b})")
        if self.kind not in ("uniform", "gaussian"):
            raise ConfigError(f"unknown disturbance kind {self.kind!r}")
        object.__setattr__(self, "ranges", rr)
        # the model is immutable: lo and span are built once (read-only arrays)
        lo = np.array([a for a, _ in rr], dtype=np.float64)
        span = np.array([b - a for a, b in rr], dtype=np.float64)  # disturbance.py:193
        lo.flags.writeable = False
        span.flags.writeable = False
        object.__setattr__(self, "_lo", lo)
        object.__setattr__(self, "_span", span)

    @property
    def state_dim(self) -> int:
        return len(self.ranges)

    @property
    def lo(self) -> np.ndarray:
        return self._lo

    @property
    def span(self) -> np.ndarray:
        # hi - lo rounded as the reference computes it (disturbance.py:193)
        return self._span

    @classmethod
    def scaled(cls, magnitude: float, state_dim: int) -> "DisturbanceModel":
        return cls(tuple((-magnitude, magnitude) for _ in range(state_dim)))


class ScenarioSet:
    """(n_sim, horizon, n) additive disturbances: dense, or generated on demand.

    Dense: ``ScenarioSet(data, seed=None, model=None)`` like the reference.
    Generated: ``ScenarioSet.generated(model, n_sim, horizon, seed, k0=0)``;
    entry (k, j, i) is the counter-RNG value at scenario index k0 + k.
    """

    __slots__ = ("_data", "seed", "model", "_n_sim", "_horizon", "k0", "device", "_stream")

    def __init__(self, data=None, seed=None, model=None):
        d = np.asarray(data, dtype=np.float64)
        if d.ndim != 3:
            raise ConfigError(f"scenario data must be 3-D (n_sim, horizon, n), got {d.shape}")
        if not np.all(np.isfinite(d)):
            raise ConfigError("scenario data must be finite")
        self._data = d
        self.seed = seed
        self.model = model
        self._n_sim, self._horizon = d.shape[0], d.shape[1]
        self.k0 = 0
        self.device = 0
        self._stream = None

    @classmethod
    def generated(cls, model: DisturbanceModel, n_sim: int, horizon: int, seed: int,
                  k0: int = 0, device: int = 0) -> "ScenarioSet":
        obj = cls.__new__(cls)
        obj._data = None
        obj.seed = int(seed)
        obj.model = model
        obj._n_sim = int(n_sim)
        obj._horizon = int(horizon)
        obj.k0 = int(k0)
        obj.device = int(device)
        obj._stream = None
        return obj

    @property
    def is_generated(self) -> bool:
        return self._data is None

    @property
    def data(self) -> np.ndarray:
        if self._data is None:
            from ._capi import context

            m = self.model
            self._data = context(self.device).sample(self.seed, self.k0, self._n_sim,
                                                     self._horizon, m.lo, m.span)
        return self._data

    scenarios = data

    @property
    def n_sim(self) -> int:
        return self._n_sim

    @property
    def horizon(self) -> int:
        return self._horizon

    @property
    def state_dim(self) -> int:
        return self.model.state_dim if self._data is None else self._data.shape[2]

    def prefix(self, n_sim: int) -> "ScenarioSet":
        """The nested subset of the first n_sim scenarios (disturbance.py:172-176)."""
        if not 1 <= n_sim <= self.n_sim:
            raise ConfigError(f"prefix size {n_sim} out of range [1, {self.n_sim}]")
        if self._data is None:
            return ScenarioSet.generated(self.model, n_sim, self._horizon, self.seed, self.k0,
                                         self.device)
        return ScenarioSet(self._data[:n_sim], seed=self.seed, model=self.model)

    def shard(self, rank: int, world: int) -> "ScenarioSet":
        """Contiguous scenario range of one rank: [k0 + rank*n/world, k0 + (rank+1)*n/world)."""
        a = rank * self.n_sim // world
        b = (rank + 1) * self.n_sim // world
        if self._data is None:
            return ScenarioSet.generated(self.model, b - a, self._horizon, self.seed,
                                         self.k0 + a, self.device)
        return ScenarioSet(self._data[a:b], seed=self.seed, model=self.model)

    def __eq__(self, other):
        if not isinstance(other, ScenarioSet):
            return NotImplemented
        return self.seed == other.seed and np.array_equal(self.data, other.data)

    __hash__ = None


def sample_scenarios(model: DisturbanceModel, n_sim: int, horizon: int, seed: int,
                     device: int = 0) -> ScenarioSet:
    """The reference's sample_scenarios (disturbance.py:179-203), generated lazily on the
    device; pass horizon = j_star + 1 for a j_star-step prediction."""
    if n_sim < 1 or horizon < 1:
        raise ConfigError(f"n_sim and horizon must be >= 1, got {n_sim}, {horizon}")
    if model.kind != "uniform":
        raise ConfigError(f"disturbance kind {model.kind!r} is reserved but not implemented")
    if model.state_dim > 16:
        raise ConfigError("at most 16 disturbance components are supported")
    return ScenarioSet.generated(model, n_sim, horizon, seed, 0, device)


def zero_scenarios(n: int, horizon: int) -> ScenarioSet:
    """The single all-zero scenario (disturbance.py:206-210)."""
    if n < 1 or horizon < 1:
        raise ConfigError(f"n and horizon must be >= 1, got {n}, {horizon}")
    return ScenarioSet(np.zeros((1, horizon, n), dtype=np.float64), seed=None)
