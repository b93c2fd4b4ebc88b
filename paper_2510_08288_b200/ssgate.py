"""The steady-state gate as an exact setpoint interval.

The reference admits a candidate setpoint v only if the tightened constraint
set contains its steady-state output, ``tight.contains(np.tanh(v))``
(governor.py:302 and 401, dynamics.py:243-244) -- evaluated with *numpy's*
tanh, which differs from glibc's in about 29% of inputs.  The device never
evaluates that tanh.  Instead the host computes, once per tightened set, the
exact set of doubles v that pass:

    {v : lo <= np.tanh(v) <= hi} = [v_lo, v_hi]

by bisection over the ordered bit patterns of doubles with numpy's own tanh,
and then *verifies* the step structure on a window of +-WINDOW ulps around
each threshold (numpy's tanh is monotone there, but the verification, not an
assumption, is what makes the gate exact).  The device then compares v
against two doubles.  Because the interval depends only on the tightened set,
it is computed once per configuration, not per step.
"""

from __future__ import annotations

import functools
import math

import numpy as np

from .errors import RefgovError

WINDOW = 4096
_SIGN = np.int64(-0x8000000000000000)


def _key(x: float) -> int:
    """Order-preserving map double -> int (ascending doubles -> ascending ints)."""
    i = int(np.array(x, dtype=np.float64).view(np.int64))
    return i if i >= 0 else -(i & 0x7FFFFFFFFFFFFFFF)


def _unkey(k: np.ndarray | int):
    k = np.asarray(k, dtype=np.int64)
    bits = np.where(k >= 0, k, (-k) | _SIGN)
    return bits.astype(np.int64).view(np.float64)


_KMAX = _key(np.finfo(np.float64).max)


def _first_true(pred, lo_key: int, hi_key: int) -> int | None:
    """Smallest key in [lo_key, hi_key] with pred True, assuming False..True."""
    if not pred(float(_unkey(hi_key))):
        return None
    if pred(float(_unkey(lo_key))):
        return lo_key
    lo, hi = lo_key, hi_key  # pred(lo) False, pred(hi) True
    while hi - lo > 1:
        mid = lo + (hi - lo) // 2
        if pred(float(_unkey(mid))):
            hi = mid
        else:
            lo = mid
    return hi


def _verify_step(pred_vec, k: int, rising: bool) -> None:
    ks = np.arange(max(k - WINDOW, -_KMAX), min(k + WINDOW, _KMAX) + 1, dtype=np.int64)
    vals = pred_vec(_unkey(ks))
    want = ks >= k if rising else ks <= k
    if not np.array_equal(vals, want):
        raise RefgovError("numpy tanh is not monotone around the steady-state threshold; "
                          "the device gate would not be exact")


@functools.lru_cache(maxsize=64)
def admissible_setpoints(ss_lower: float, ss_upper: float) -> tuple[float, float]:
    """[v_lo, v_hi] with ss_lower <= np.tanh(v) <= ss_upper  <=>  v_lo <= v <= v_hi.

    Returns (inf, -inf) when no double passes.  Infinite outer ends mean the
    bound never binds.
    """
    lo_pred = lambda v: bool(np.tanh(np.float64(v)) >= ss_lower)  # noqa: E731
    hi_pred = lambda v: bool(np.tanh(np.float64(v)) > ss_upper)   # noqa: E731
    k_lo = _first_true(lo_pred, -_KMAX, _KMAX)
    if k_lo is None:
        return math.inf, -math.inf
    k_hi_excl = _first_true(hi_pred, -_KMAX, _KMAX)
    k_hi = _KMAX if k_hi_excl is None else k_hi_excl - 1
    if k_hi < k_lo:
        return math.inf, -math.inf
    if k_lo > -_KMAX:
        _verify_step(lambda v: np.tanh(v) >= ss_lower, k_lo, rising=True)
        v_lo = float(_unkey(k_lo))
    else:
        v_lo = -math.inf
    if k_hi < _KMAX:
        _verify_step(lambda v: np.tanh(v) <= ss_upper, k_hi, rising=False)
        v_hi = float(_unkey(k_hi))
    else:
        v_hi = math.inf
    return v_lo, v_hi


def gate(v: float, interval: tuple[float, float]) -> bool:
    return interval[0] <= v <= interval[1]
