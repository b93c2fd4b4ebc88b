"""The library's restatement of numpy's float64 tanh (rg_nptanh.h, numpy 2.3.5's SIMD
kernel) and the surrogate true-plant step built on it, against numpy itself -- the host
arithmetic of the native closed loop (rg_closed_loop).  Host code: no device needed."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2510_08288_b200 import _capi
from paper_2510_08288_b200.dynamics import _surrogate_rk4


def _inputs(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    parts = [rng.uniform(-30, 30, n), rng.uniform(-2, 2, n), rng.standard_normal(n),
             (10.0 ** rng.uniform(-300, 1.6, n // 2)) * rng.choice([-1, 1], n // 2)]
    # +-300 ulps around every interval boundary (0.1875 * 2^k and 0.28125 * 2^k, up to 24)
    edges = [0.1875 * 2.0 ** e * m for e in range(-3, 7) for m in (1.0, 1.5)]
    edges = np.array(sorted({s * v for v in edges for s in (1.0, -1.0)}))
    near = (edges[:, None].view(np.int64) + np.arange(-300, 301)[None, :]).ravel()
    special = np.array([0.0, -0.0, 5e-324, -5e-324, 1e-310, 24.0, -24.0, 1e300, -1e300,
                        np.nextafter(24.0, 0.0), np.nextafter(0.1875, 0.0)])
    return np.concatenate(parts + [near.view(np.float64), special])


def test_np_tanh_is_numpys_bit_for_bit():
    x = _inputs(500_000, 11)
    got = _capi.np_tanh(x)
    ref = np.tanh(x)
    bad = np.flatnonzero(got.view(np.uint64) != ref.view(np.uint64))
    assert bad.size == 0, (x[bad[:5]], got[bad[:5]], ref[bad[:5]])


@pytest.mark.parametrize("h", [0.01, 0.05])
def test_plant_step_equals_the_python_plant(h):
    """rg_plant_step = dynamics._surrogate_rk4 (the reference's elementwise RK4 with numpy
    tanh), state and setpoint over the operating box and beyond."""
    rng = np.random.default_rng(int(h * 1000))
    for _ in range(3000):
        x = rng.uniform(-3, 3, 3) * rng.choice([1e-3, 1.0, 10.0])
        v = float(rng.uniform(-3, 3))
        got = _capi.plant_step(h, x, v)
        ref = _surrogate_rk4(h, x, v)
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), (x, v, got, ref)
