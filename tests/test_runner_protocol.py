"""The file-protocol runner (reference backend_gpu.py:9-18, 50-140).

A client written here plays the reference's backend_gpu.fill: it writes the
RGSC dump and request.json, runs the runner as a subprocess and reads p.bin and
response.json back.  On a B200 the matrix must equal the CPU oracle's on the
same (float32-rounded) scenarios bit for bit.
"""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2510_08288_b200 as rg
from paper_2510_08288_b200.runner import read_rgsc, write_rgsc

ROOT = Path(__file__).resolve().parents[1]


def _request(tmp, x0, v_rows, dist, j_star, lower, upper, ss_lower, ss_upper):
    write_rgsc(tmp / "scenarios.rgsc", dist)
    req = {"plant": {"kind": "surrogate-fc", "step_size": 0.01}, "x0": [float(a) for a in x0],
           "v_rows": [float(v) for v in v_rows], "j_star": int(j_star),
           "bounds": {"lower": lower, "upper": upper},
           "ss_bounds": {"lower": ss_lower, "upper": ss_upper},
           "scenarios": str(tmp / "scenarios.rgsc"), "p_out": str(tmp / "p.bin"),
           "response": str(tmp / "response.json")}
    (tmp / "request.json").write_text(json.dumps(req))
    return subprocess.run([sys.executable, "-m", "paper_2510_08288_b200.runner",
                           str(tmp / "request.json")], cwd=str(ROOT), capture_output=True,
                          text=True, timeout=300)


def test_rgsc_round_trip_is_float32(tmp_path):
    d = np.random.default_rng(0).uniform(-1, 1, (3, 5, 3))
    write_rgsc(tmp_path / "x.rgsc", d)
    back = read_rgsc(tmp_path / "x.rgsc")
    assert back.shape == d.shape
    assert np.array_equal(back, d.astype(np.float32).astype(np.float64))
    raw = (tmp_path / "x.rgsc").read_bytes()
    assert raw[:4] == b"RGSC" and len(raw) == 16 + 4 * d.size


def test_runner_reports_failure_through_the_protocol(tmp_path):
    dist = np.zeros((2, 9, 3))
    req = {"plant": {"kind": "linear-oracle"}, "x0": [0, 0, 0], "v_rows": [0.1], "j_star": 8,
           "bounds": {"lower": -0.9, "upper": 0.9}, "ss_bounds": {"lower": None, "upper": None},
           "scenarios": str(tmp_path / "s.rgsc"), "p_out": str(tmp_path / "p.bin"),
           "response": str(tmp_path / "r.json")}
    write_rgsc(tmp_path / "s.rgsc", dist)
    (tmp_path / "q.json").write_text(json.dumps(req))
    r = subprocess.run([sys.executable, "-m", "paper_2510_08288_b200.runner",
                        str(tmp_path / "q.json")], cwd=str(ROOT), capture_output=True, text=True)
    assert r.returncode == 1
    resp = json.loads((tmp_path / "r.json").read_text())
    assert resp["ok"] is False and "unsupported plant" in resp["error"]


@pytest.mark.gpu
def test_runner_fill_equals_oracle_on_protocol_data(tmp_path, orc):
    rng = np.random.default_rng(5)
    n, j_star, m = 40, 128, 16
    v_prev, r = 0.3, 2.4
    x0 = np.array([np.tanh(v_prev), v_prev, np.tanh(v_prev) / 2]) + 0.02
    dist64 = rg.sample_scenarios(rg.DisturbanceModel.scaled(0.02, 3), n, j_star + 1, 3).data
    grid = rg.grid_kappas(m)
    v_rows = np.array([rg.update_setpoint(v_prev, r, float(k)) for k in grid])
    tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
    out = _request(tmp_path, x0, v_rows, dist64, j_star, -0.9, 0.9, tight.lower, tight.upper)
    assert out.returncode == 0, out.stderr
    resp = json.loads((tmp_path / "response.json").read_text())
    assert resp["ok"] is True
    P = np.frombuffer((tmp_path / "p.bin").read_bytes(), dtype=np.uint8).reshape(m, n)
    dist32 = dist64.astype(np.float32).astype(np.float64)
    P_ref, _, _, _ = orc.fill_feasibility(0.01, x0, v_prev, r, grid, dist32, -0.9, 0.9,
                                          tight.lower, tight.upper, j_star)
    assert np.array_equal(P.astype(bool), P_ref)
    assert 0 < P.sum() < P.size   # the case binds
