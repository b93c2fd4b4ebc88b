"""Time the reference's OWN API driving the device (one B200), at C2 (1000 scenarios, j* = 256,
M = 32, bench snapshot), scenarios presampled by the reference (its kernel-only mode):

  plugin     refgov.robust_rg_parallel(backend="cuda") after refgov_plugin.install (in process;
             the reference's dense host tensor goes through pinned staging into rg_fill)
  gpu-seam   refgov.robust_rg_parallel(backend="gpu") with the plugin's in-process backend_gpu.fill
  runner     refgov.robust_rg_parallel(backend="gpu") through REFGOV_GPU_RUNNER (the reference's
             subprocess + temp-file protocol, one process start per call: backend_gpu.py:50-140)
  multicore  the reference's own multicore backend, for scale
Prints one JSON object.  Uses the reference staged in oracle/_ref (test infrastructure)."""
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from oracle import reference  # noqa: E402
from paper_2510_08288_b200 import refgov_plugin  # noqa: E402

rf, why = reference.load()
assert rf is not None, why
plant = rf.make_plant("surrogate-fc")
box = rf.ConstraintSet(-0.9, 0.9, anchor=0.0)
scen = [rf.sample_scenarios(rf.DisturbanceModel.scaled(0.001, 3), 1000, 257, seed=7 + q)
        for q in range(4)]


def timed(backend, reps):
    cfg = rf.GovernorConfig(j_star=256, m_grid=32, n_sim=1000, backend=backend)
    rf.robust_rg_parallel(plant, np.zeros(3), rf.GovernorState(0.0), 0.5, box, scen[0], cfg)
    ts = []
    for q in range(reps):
        t0 = time.perf_counter()
        r = rf.robust_rg_parallel(plant, np.zeros(3), rf.GovernorState(0.0), 0.5, box,
                                  scen[q % 4], cfg)
        ts.append((time.perf_counter() - t0) * 1e3)
        assert r.kappa_opt == 1.0 and r.matrix.all()
    return {"ms_median": statistics.median(ts), "ms_min": min(ts), "reps": reps,
            "backend_stat": r.diagnostics.get("backend")}


out = {"workload": "C2 bench snapshot, 1000 scenarios x 32 candidates x 256 steps, presampled",
       "multicore": timed("multicore", 10)}
refgov_plugin.install(rf)
out["plugin_cuda"] = timed("cuda", 50)
out["gpu_seam_in_process"] = timed("gpu", 50)
refgov_plugin.uninstall(rf)
os.environ["REFGOV_GPU_RUNNER"] = f"{sys.executable} -m paper_2510_08288_b200.runner"
os.environ["PYTHONPATH"] = str(ROOT) + os.pathsep + os.environ.get("PYTHONPATH", "")
out["runner_protocol"] = timed("gpu", 3)
print(json.dumps(out))
