"""Host plant mirror (paper_2510_08288_b200/dynamics.py): the reference's known answers.

CPU-only.  Restates the surrogate/linear plant checks of the reference's
`pkg/tests/test_dynamics.py:80-110` for the host-side plant the closed loop uses
as the true plant (numpy tanh, as the reference), and pins its step against
the oracle's restatement of `dynamics.py:110-130, 228-231`.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2510_08288_b200 as rg


def test_surrogate_steady_state_is_saturating():
    plant = rg.make_plant("surrogate-fc")
    assert plant.steady_state_output(0.0) == 0.0
    assert plant.steady_state_output(1.0) == np.tanh(1.0)
    assert abs(plant.steady_state_output(50.0)) < 1.0 + 1e-12


def test_surrogate_converges_to_equilibrium():
    plant = rg.make_plant("surrogate-fc")
    x, v = np.zeros(3), 0.8
    for _ in range(2000):
        x = plant.step(x, v)
    assert plant.output(x, v) == pytest.approx(np.tanh(v), abs=1e-6)


def test_surrogate_equilibrium_is_fixed_point():
    plant = rg.make_plant("surrogate-fc")
    v = 1.3
    xeq = np.array([np.tanh(v), v, np.tanh(v) / 2.0])
    assert plant.step(xeq, v) == pytest.approx(xeq, abs=1e-12)


def test_host_step_equals_oracle_restatement(orc):
    plant = rg.make_plant("surrogate-fc")
    rng = np.random.default_rng(12)
    for _ in range(200):
        x = rng.uniform(-2.0, 2.0, 3)
        v = float(rng.uniform(-3.0, 3.0))
        assert np.array_equal(plant.step(x, v), orc.plant_step(0.01, x, v))


def test_overflow_reports_state_index():
    plant = rg.make_plant("surrogate-fc", step_size=1.0)
    with pytest.raises(rg.IntegrationOverflowError) as exc:
        plant.step(np.zeros(3), 1e7)          # x2 is driven past the 1e6 box
    assert exc.value.state_index == 1


def test_linear_plant_validation():
    with pytest.raises(rg.ConfigError):
        rg.LinearOraclePlant([[1.0]], [1.0], [1.0])          # spectral radius 1
    with pytest.raises(rg.ConfigError):
        rg.make_plant("linear-oracle", A=[[0.5]])           # B, C missing
    plant = rg.make_plant("linear-oracle", A=[[0.5]], B=[0.5], C=[1.0])
    assert plant.steady_state_output(2.0) == pytest.approx(2.0)
    x = np.zeros(1)
    ys = []
    for _ in range(4):
        ys.append(plant.output(x, 1.0))
        x = plant.step(x, 1.0)
    assert ys == pytest.approx([0.0, 0.5, 0.75, 0.875])   # test_dynamics.py step response


def test_scalar_surrogate_step_equals_array_form_and_reference():
    """The closed loop's true-plant step in Python floats (one numpy tanh call for the four
    stage arguments) equals the 3-element numpy form of dynamics.py:110-130 bit for bit --
    and the unmodified reference's plant.step when it is staged (oracle/_ref) -- including
    the overflow abort."""
    import numpy as np

    import paper_2510_08288_b200 as rg
    from paper_2510_08288_b200 import dynamics as D
    from oracle import reference

    p = rg.make_plant("surrogate-fc")
    ref, _ = reference.load()
    rp = ref.make_plant("surrogate-fc") if ref is not None else None
    rng = np.random.default_rng(5)
    X = np.concatenate([rng.uniform(-1, 1, (3000, 3)), rng.uniform(-40, 40, (1000, 3)),
                        rng.uniform(-9e5, 9e5, (500, 3))])
    V = rng.uniform(-3, 3, X.shape[0])
    for i in range(X.shape[0]):
        a = D.rk4_step(p, X[i], float(V[i]))
        b = p.step(X[i], float(V[i]))
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), i
        if rp is not None and i % 7 == 0:
            c = rp.step(X[i], float(V[i]))
            assert np.array_equal(c.view(np.uint64), b.view(np.uint64)), i
    import pytest
    for bad in ([1e300, 0.0, 0.0], [0.0, 0.0, 2e6]):
        with pytest.raises(rg.IntegrationOverflowError) as e1:
            D.rk4_step(p, np.array(bad), 0.1)
        with pytest.raises(rg.IntegrationOverflowError) as e2:
            p.step(np.array(bad), 0.1)
        assert e1.value.state_index == e2.value.state_index
