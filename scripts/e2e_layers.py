"""Host cost of the public grid-step API at C2, layer by layer (1000 calls each, median of
5 repetitions): the raw C call, the ctypes wrapper (Context.grid_step), robust_rg_parallel
with P returned, and sample_scenarios + robust_rg_parallel (bench.py's e2e loop)."""
import sys
import time
import numpy as np
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
from paper_2510_08288_b200.governor import _prepared, _source

plant = rg.make_plant("surrogate-fc")
box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
model = rg.DisturbanceModel.scaled(0.001, 3)
cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=1000)
ctx = _capi.context(0)
prob = _prepared(0.01, -0.9, 0.9, 0.0, 0.05, "scale", 256, 32)[0]
scen = rg.sample_scenarios(model, 1000, 257, seed=5, device=0)
_, _, stream = _source(scen, 256)
x0 = np.zeros(3)
res = _capi.GridResult()
pb = np.empty((32, 32), dtype=np.uint32)


def raw():
    _capi.check(ctx.lib.rg_grid_step(ctx.handle, prob, x0.ctypes.data, 0.0, 0.5, 32, 0, None,
                                     1000, 0, stream, None, pb.ctypes.data, res, _capi.RG_NO_TIMING))


def wrapper():
    ctx.grid_step(prob, x0, 0.0, 0.5, 32, False, None, 1000, stream, True, timing=False,
                  want_viol=False)


def api():
    rg.robust_rg_parallel(plant, x0, rg.GovernorState(0.0), 0.5, box, scen, cfg)


def api_sample():
    s = rg.sample_scenarios(model, 1000, 257, seed=11, device=0)
    rg.robust_rg_parallel(plant, x0, rg.GovernorState(0.0), 0.5, box, s, cfg)


for name, f in (("raw C call", raw), ("ctypes wrapper", wrapper), ("robust_rg_parallel", api),
                ("sample + robust_rg_parallel", api_sample)):
    for _ in range(50):
        f()
    reps = []
    for _ in range(5):
        t0 = time.perf_counter()
        for _ in range(1000):
            f()
        reps.append((time.perf_counter() - t0) / 1000 * 1e6)
    print(f"{name:30s} {np.median(reps):8.1f} us per call", flush=True)
