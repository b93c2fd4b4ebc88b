"""bench.py's driver contract on the CPU: the reference arm's JSON line (it runs
the oracle port on the host) and the issue-bound model's arithmetic."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1", "--n-sim", "200"],
                         capture_output=True, text=True, check=True, timeout=300)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["steps"] == 2 and d["higher_is_better"] is True
    # the unmodified reference (oracle/_ref, numba) when staged, else the oracle's C port
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] == d["e2e"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C2 bench snapshot")
    assert d["config"]["n_sim"] == 200


def test_config_is_shared_by_both_arms():
    """Both arms print the same config dict (the driver's same_config check)."""
    sys.path.insert(0, str(ROOT))
    import bench

    for wl in ("c1", "c2", "c3", "c4", "c5"):
        spec = dict(bench.WORKLOADS[wl])
        a = bench.config_of(wl, spec, 4, 256)
        b = bench.config_of(wl, dict(spec), 4, 256)
        assert a == b and a["workload"] == spec["name"]
    assert bench.config_of("c4", dict(bench.WORKLOADS["c4"]), 8, 256)["n_sim"] == 1 << 20


def test_gpus_flag_must_match_world_size():
    env = dict(**__import__("os").environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--impl",
                          "reference", "--steps", "1"], capture_output=True, text=True, env=env,
                         timeout=120)
    assert out.returncode == 2 and "WORLD_SIZE=2" in out.stderr


def test_active_cells_matches_host_rows():
    """C5's work count (the reference's sims_run / n_sim per episode) against the
    product's own host gate + dedup loop (governor._host_rows)."""
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2510_08288_b200.governor import _host_rows, grid_kappas

    rng = __import__("numpy").random.default_rng(0)
    import numpy as np
    E = 300
    vp = np.concatenate([rng.uniform(-1.5, 1.5, E - 50), np.full(50, 0.4)])
    r = np.concatenate([rng.uniform(-2.5, 2.5, E - 100), np.full(50, 0.4), np.full(50, 2.5)])
    interval = (-1.27, 1.27)
    got = bench.active_cells(vp, r, 32, interval)
    grid = grid_kappas(32).tolist()
    for e in range(E):
        _, _, _, reps = _host_rows(float(vp[e]), float(r[e]), grid, interval)
        assert got[e] == len(reps), e


def test_issue_model_arithmetic():
    sys.path.insert(0, str(ROOT))
    import bench

    m = bench.issue_model(1000, 256, 1.0, {"sm_mhz": 1965.0})
    ncu = bench._ncu_summary()
    fp64, total = ncu["fp64_instr_per_cell_step"], ncu["instr_per_cell_step"]
    assert abs(m["cycles_per_warp_step"] - (2 * fp64 + (total - fp64))) < 1e-9
    warp_steps = 32 * 32 * 256  # ceil(1000/32) warps per row, 32 rows, 256 steps
    assert abs(m["bound_ms"] - warp_steps / 592 * m["cycles_per_warp_step"] / 1965e3) < 1e-12
    assert abs(m["frac"] - m["bound_ms"]) < 1e-12  # measured 1 ms
    # above one wave the multi-wave form's counts are used
    big = bench.issue_model(1 << 20, 256, 100.0, {"sm_mhz": 1965.0})
    ncu10k = bench._ncu_summary("k_grid_ncu_10k.json")
    assert abs(big["cycles_per_warp_step"] - (ncu10k["fp64_instr_per_cell_step"]
                                              + ncu10k["instr_per_cell_step"])) < 1e-9


def test_reference_arm_c1_line():
    """C1's reference arm: the reference's own bisection loop on one host core (when the
    reference is staged; the C port has no closed-loop driver and reports value None)."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--workload", "c1", "--cpu-seconds", "2"],
                         capture_output=True, text=True, check=True, timeout=600)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["config"]["workload"].startswith("C1")
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] == 1
    if cb["kind"] == "reference":
        assert d["value"] == cb["value"] > 0 and d["ms_per_step"] > 0
