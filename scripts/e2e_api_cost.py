"""Where the public-API grid step (bench.py's e2e) spends its time at C2, piece by piece."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2510_08288_b200 as rg  # noqa: E402
from paper_2510_08288_b200 import _capi, governor as G  # noqa: E402

N = 500


def timeit(name, fn):
    for _ in range(30):
        fn()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    dt = (time.perf_counter() - t0) / N * 1e6
    print(f"{name:58s} {dt:8.1f} us", flush=True)
    return dt


plant = rg.make_plant("surrogate-fc")
box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
model = rg.DisturbanceModel.scaled(0.001, 3)
cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=1000)
x0 = np.zeros(3)
scen = rg.sample_scenarios(model, 1000, 257, seed=7)
ctx = _capi.context(0)
lib = ctx.lib

timeit("sample_scenarios (descriptor)", lambda: rg.sample_scenarios(model, 1000, 257, seed=7))
timeit("robust_rg_parallel, P kept (bench e2e minus sampling)", lambda: rg.robust_rg_parallel(
    plant, x0, rg.GovernorState(0.0), 0.5, box, scen, cfg))
cfg2 = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=1000, keep_matrix=False)
timeit("robust_rg_parallel, no P", lambda: rg.robust_rg_parallel(
    plant, x0, rg.GovernorState(0.0), 0.5, box, scen, cfg2))
prob, iv, grid, grid_list = G._prepared(0.01, -0.9, 0.9, 0.0, 0.05, "scale", 256, 32)
timeit("_prepared (cached)", lambda: G._prepared(0.01, -0.9, 0.9, 0.0, 0.05, "scale", 256, 32))
timeit("_source", lambda: G._source(scen, 256))
dist, n_sim, stream = G._source(scen, 256)
timeit("ctx.grid_step with pbits (zero-copy, sync)", lambda: ctx.grid_step(
    prob, x0, 0.0, 0.5, 32, False, dist, n_sim, stream, want_pbits=True, abandon=False,
    timing=False, want_viol=False))
timeit("ctx.grid_step no pbits", lambda: ctx.grid_step(
    prob, x0, 0.0, 0.5, 32, False, dist, n_sim, stream, want_pbits=False, abandon=True,
    timing=False, want_viol=False))
res = _capi.GridResult()
x0p = x0.ctypes.data_as(ctypes.c_void_p)
timeit("raw ctypes rg_grid_step (sync, no pbits, no timing)", lambda: lib.rg_grid_step(
    ctx.handle, ctypes.byref(prob), x0p, 0.0, 0.5, 32, 0, None, 1000, 0, ctypes.byref(stream),
    None, None, ctypes.byref(res), _capi.RG_NO_TIMING))
pb = np.zeros((32, 32), np.uint32)
timeit("np.unpackbits of P", lambda: np.unpackbits(pb.view(np.uint8), axis=1,
                                                   bitorder="little")[:, :1000].view(np.bool_))
r = rg.robust_rg_parallel(plant, x0, rg.GovernorState(0.0), 0.5, box, scen, cfg)
print("kernel_us", r.diagnostics["kernel_us"])
