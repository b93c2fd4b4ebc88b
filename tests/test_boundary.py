"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every
symbol include/refgov_b200.h declares, the ctypes structs match the header's
layout, the host-side gate is exact, and errors without a device are loud."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
from paper_2510_08288_b200.ssgate import admissible_setpoints

HEADER = Path(__file__).resolve().parents[1] / "include" / "refgov_b200.h"


def _declared():
    return re.findall(r"^RG_API [^(]*?\b(rg_\w+)\(", HEADER.read_text(), flags=re.M)


def test_library_exports_every_declared_symbol():
    lib = _capi.load_library()
    names = _declared()
    assert len(names) >= 15
    assert set(names) == set(_capi.SIGNATURES)
    for n in names:
        assert hasattr(lib, n), n
    assert lib.rg_abi_version() == 1


def test_struct_layouts_match_header():
    # sizes of the C structs, computed from their field lists in the header
    assert ctypes.sizeof(_capi.Problem) == 5 * 8 + 2 * 4
    assert ctypes.sizeof(_capi.Scenarios) == 8 * 3 + 8 * 8
    assert ctypes.sizeof(_capi.LinearPlant) == 8 + 8 * (16 + 4 + 4 + 4)
    assert ctypes.sizeof(_capi.GridResult) == 4 * 4 + 4 * 8 + 4 + 4
    assert ctypes.sizeof(_capi.BisectResult) == 8 + 4 + 4 + 8 + 8 + 4 + 4


def test_no_device_is_a_loud_error():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except ImportError:
        pass
    with pytest.raises(rg.BackendUnavailableError):
        _capi.Context(0)
    with pytest.raises(rg.BackendUnavailableError):
        rg.robust_rg_parallel(rg.make_plant("surrogate-fc"), np.zeros(3), rg.GovernorState(),
                              0.5, rg.ConstraintSet(-0.9, 0.9), rg.zero_scenarios(3, 33),
                              rg.GovernorConfig(j_star=32, n_sim=1))


@pytest.mark.parametrize("lo,hi", [(-0.855, 0.855), (-0.45, 0.855), (-np.inf, 0.855),
                                   (-0.2, np.inf), (0.1, 0.3), (-0.999, 0.9999999)])
def test_ss_interval_equals_numpy_gate(lo, hi):
    v_lo, v_hi = admissible_setpoints(lo, hi)
    rng = np.random.default_rng(1)
    v = np.concatenate([rng.uniform(-6, 6, 200_000),
                        v_lo + rng.integers(-5000, 5000, 20_000) * np.spacing(v_lo)
                        if np.isfinite(v_lo) else np.zeros(0),
                        v_hi + rng.integers(-5000, 5000, 20_000) * np.spacing(v_hi)
                        if np.isfinite(v_hi) else np.zeros(0)])
    y = np.tanh(v)
    numpy_gate = (y >= lo) & (y <= hi)
    interval_gate = (v >= v_lo) & (v <= v_hi)
    assert np.array_equal(numpy_gate, interval_gate)


def test_ss_interval_covers_every_dyadic_candidate():
    """Every setpoint bisection can test in the golden cases gates identically."""
    tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
    iv = admissible_setpoints(tight.lower, tight.upper)
    rng = np.random.default_rng(3)
    for _ in range(200):
        v_prev, r = rng.uniform(-2, 2), rng.uniform(-3, 3)
        for m in range(0, 257):
            v = rg.update_setpoint(v_prev, r, m / 256)
            assert tight.contains(float(np.tanh(v))) == (iv[0] <= v <= iv[1])


def test_host_mirrors_match_oracle(orc):
    for z in (0, 1, 2**63, 2**64 - 1, 123456789):
        assert rg.splitmix64(z) == orc.splitmix64(z)
    assert rg.derive_seed(2024, "scenarios") == orc.derive_seed(2024, "scenarios")
    assert rg.counter_uniform(7, 3, 2, 1) == orc.counter_uniform(7, 3, 2, 1)
    assert rg.update_setpoint(0.1, 0.30000000000000004, 1.0) == 0.30000000000000004
    with pytest.raises(rg.DomainError):
        rg.update_setpoint(0.0, 1.0, 1.01)
    P = np.array([[1], [0], [1]], dtype=bool)
    assert rg.extract_kappa_opt(P) == (3, 1.0)
    assert rg.extract_kappa_opt(P, prefix_mode=True) == (1, 0.0)
    assert rg.extract_kappa_opt(np.zeros((4, 3), bool)) == (None, None)


def test_config_validation_mirrors_reference():
    for bad in (dict(epsilon=0.0), dict(epsilon=1.0), dict(m_grid=1), dict(n_kappa=0),
                dict(n_sim=0), dict(backend="tpu"), dict(backend="serial"),
                dict(infeasible_policy="panic"), dict(tighten_mode="shrink"),
                dict(tighten_mode="margin", epsilon=0.0), dict(workers=0)):
        with pytest.raises(rg.ConfigError):
            rg.GovernorConfig(**bad)
    rg.GovernorConfig(tighten_mode="margin", epsilon=1.5)
    rg.GovernorConfig(backend="gpu")


def test_first_context_in_fresh_process_does_not_hang():
    """context() before any other library call (regression: lock re-entry deadlock)."""
    import subprocess
    import sys

    code = ("import paper_2510_08288_b200 as rg\n"
            "from paper_2510_08288_b200 import _capi\n"
            "try:\n    _capi.context(0)\nexcept rg.BackendUnavailableError:\n    pass\n")
    r = subprocess.run([sys.executable, "-c", code], timeout=120,
                       cwd=str(Path(__file__).resolve().parents[1]))
    assert r.returncode == 0


def test_host_rows_match_reference_gate_and_dedup():
    """governor._host_rows (vectorised v_rows, interval gate, dedup) equals the
    reference's per-row loop with numpy tanh and a dict (governor.py:286-317)."""
    from paper_2510_08288_b200.governor import _host_rows, _prepared

    plant = rg.make_plant("surrogate-fc")
    tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
    _, iv, g, _ = _prepared(0.01, -0.9, 0.9, 0.0, 0.05, "scale", 256, 32)
    rng = np.random.default_rng(1)
    for trial in range(1500):
        vp = float(rng.choice([rng.uniform(-2, 2), 0.3, -0.0, 1.2744531163104806]))
        r = float(rng.choice([rng.uniform(-3, 3), vp, 2.5, np.nextafter(vp, 9)]))
        grid = g if trial % 2 else np.sort(rng.uniform(0, 1, 17))
        v, ok, dup, reps = _host_rows(vp, r, grid.tolist(), iv)
        v = np.array(v)
        v_ref = [rg.update_setpoint(vp, r, float(k)) for k in grid]
        ok_ref = [tight.contains(plant.steady_state_output(x)) for x in v_ref]
        first, dup_ref, reps_ref = {}, [-1] * len(grid), []
        for i in range(len(grid)):
            if ok_ref[i]:
                if v_ref[i] in first:
                    dup_ref[i] = first[v_ref[i]]
                else:
                    first[v_ref[i]] = i
                    reps_ref.append(i)
        assert np.array_equal(np.array(v_ref).view(np.uint64), v.view(np.uint64))
        assert list(ok) == ok_ref and list(dup) == dup_ref and list(reps) == reps_ref
