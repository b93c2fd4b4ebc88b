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
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] == d["e2e"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C2 bench snapshot")


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
