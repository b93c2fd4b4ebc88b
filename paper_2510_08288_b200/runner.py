"""Device runner speaking the reference's GPU file protocol (backend_gpu.py:9-18).

The unmodified reference package reaches a GPU by running the command in
REFGOV_GPU_RUNNER with a request file (backend_gpu.py:50-140).  Pointing it here

    REFGOV_GPU_RUNNER="python -m paper_2510_08288_b200.runner"

makes `refgov.robust_rg_parallel(..., backend="gpu")` run its feasibility fill
on the B200.  Per call the runner

  1. reads request.json (plant, x0, v_rows, j_star, bounds, ss_bounds with
     null = unbounded, paths) and the RGSC scenario dump (disturbance.py:216-242:
     "RGSC", three little-endian uint32 (n_sim, horizon, n), float32 data);
  2. rolls every (v_row, scenario) cell out on the device in FP64 (rg_fill),
     gating each row with tight.contains(np.tanh(v)) through the exact setpoint
     interval (ssgate.py) -- the values the CPU backends would produce for the
     float32-rounded scenarios the protocol carries;
  3. writes P as row-major uint8 to p_out and {"ok": true, "kernel_us",
     "total_us", "early_terms"} to the response path.

Failures write {"ok": false, "error": ...} and exit 1, which the reference maps
to BackendUnavailableError (backend_gpu.py:115-126).
"""

from __future__ import annotations

import json
import math
import struct
import sys
import time
from pathlib import Path

import numpy as np

RGSC_MAGIC = b"RGSC"


def read_rgsc(path) -> np.ndarray:
    raw = Path(path).read_bytes()
    if len(raw) < 16 or raw[:4] != RGSC_MAGIC:
        raise ValueError(f"{path}: not an RGSC file")
    n_sim, horizon, n = struct.unpack("<III", raw[4:16])
    if len(raw) != 16 + 4 * n_sim * horizon * n:
        raise ValueError(f"{path}: size does not match ({n_sim}, {horizon}, {n})")
    data = np.frombuffer(raw, dtype="<f4", offset=16).astype(np.float64)
    return data.reshape(n_sim, horizon, n)


def write_rgsc(path, data: np.ndarray) -> None:
    data = np.asarray(data)
    header = RGSC_MAGIC + struct.pack("<III", *data.shape)
    Path(path).write_bytes(header + np.ascontiguousarray(data, dtype="<f4").tobytes())


def _bound(b, default):
    return default if b is None else float(b)


def fill_rows(h, x0, v_rows, dist, j_star, lo, hi, slo, shi, device=0):
    """The runner's fill (backend_gpu.py:50-140 contract): every gated row rolled out
    against every scenario on the device, P = OK & steady-state gate.  Returns
    (P, early_terms, kernel_us)."""
    from . import _capi
    from .ssgate import admissible_setpoints

    x0 = np.asarray(x0, dtype=np.float64)
    v_rows = np.ascontiguousarray(v_rows, dtype=np.float64)
    if dist.shape[2] != 3 or x0.shape != (3,):
        raise ValueError("the surrogate plant has 3 states")
    m, n_sim = v_rows.size, dist.shape[0]
    vlo, vhi = admissible_setpoints(slo, shi)
    gate = (v_rows >= vlo) & (v_rows <= vhi)
    rows = np.flatnonzero(gate).astype(np.int32)
    ctx = _capi.context(int(device))
    prob = _capi.Problem(float(h), lo, hi, vlo, vhi, int(j_star), 0)
    S = np.zeros((m, n_sim), dtype=np.uint8)
    steps = np.zeros((m, n_sim), dtype=np.int32)
    t1 = time.perf_counter()
    ctx.fill(prob, x0, v_rows, rows, dist, n_sim, None, S, steps)
    kernel_us = int((time.perf_counter() - t1) * 1e6)
    P = (S == 1) & gate[:, None]
    early = int(np.count_nonzero(steps[rows] < j_star)) if rows.size else 0
    return P, early, kernel_us


def serve(request_path: str) -> int:
    t0 = time.perf_counter()
    req = json.loads(Path(request_path).read_text())
    resp_path = Path(req["response"])
    try:
        plant = req["plant"]
        if plant.get("kind") != "surrogate-fc":
            raise ValueError(f"unsupported plant kind {plant.get('kind')!r}")
        h = float(plant.get("step_size", 0.01))
        lo = _bound(req["bounds"]["lower"], -math.inf)
        hi = _bound(req["bounds"]["upper"], math.inf)
        slo = _bound(req["ss_bounds"]["lower"], -math.inf)
        shi = _bound(req["ss_bounds"]["upper"], math.inf)
        dist = read_rgsc(req["scenarios"])
        P, early, kernel_us = fill_rows(h, req["x0"], req["v_rows"], dist, int(req["j_star"]), lo,
                                        hi, slo, shi, int(req.get("device", 0)))
        Path(req["p_out"]).write_bytes(P.astype(np.uint8).tobytes())
        resp = {"ok": True, "kernel_us": kernel_us,
                "total_us": int((time.perf_counter() - t0) * 1e6), "early_terms": early}
        resp_path.write_text(json.dumps(resp))
        return 0
    except Exception as e:  # the protocol's error channel
        resp_path.write_text(json.dumps({"ok": False, "error": f"{type(e).__name__}: {e}"}))
        print(f"runner: {e}", file=sys.stderr)
        return 1


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    if len(argv) != 1:
        print("usage: python -m paper_2510_08288_b200.runner <request.json>", file=sys.stderr)
        return 2
    return serve(argv[0])


if __name__ == "__main__":
    sys.exit(main())
