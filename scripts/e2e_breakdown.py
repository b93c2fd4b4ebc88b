"""Where the host time of one public-API grid step goes (C2 workload)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2510_08288_b200 as rg  # noqa: E402
from paper_2510_08288_b200 import _capi, governor as G  # noqa: E402

plant = rg.make_plant("surrogate-fc")
box = rg.ConstraintSet(-0.9, 0.9)
model = rg.DisturbanceModel.scaled(0.001, 3)
cfg = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=1000)
x0 = np.zeros(3)
ctx = _capi.context(0)
N = 300


def timeit(name, fn):
    for _ in range(10):
        fn()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    print(f"{name:45s} {(time.perf_counter() - t0) / N * 1e6:8.1f} us")


scen = rg.sample_scenarios(model, 1000, 257, seed=7)
timeit("robust_rg_parallel (keep_matrix)", lambda: rg.robust_rg_parallel(
    plant, x0, rg.GovernorState(0.0), 0.5, box, scen, cfg))
cfg2 = rg.GovernorConfig(j_star=256, m_grid=32, n_sim=1000, keep_matrix=False)
timeit("robust_rg_parallel (no matrix)", lambda: rg.robust_rg_parallel(
    plant, x0, rg.GovernorState(0.0), 0.5, box, scen, cfg2))
prob, iv, grid, grid_list = G._prepared(0.01, -0.9, 0.9, 0.0, 0.05, "scale", 256, 32)
timeit("_host_rows", lambda: G._host_rows(0.0, 0.5, grid_list, iv))
timeit("_source", lambda: G._source(scen, 256))
_, n, st = G._source(scen, 256)
timeit("ctx.grid_step (pbits)", lambda: ctx.grid_step(prob, x0, 0.0, 0.5, 32, False, None, n, st,
                                                      True))
timeit("ctx.grid_step (no pbits)", lambda: ctx.grid_step(prob, x0, 0.0, 0.5, 32, False, None, n,
                                                         st, False))
res, viol, pbits = ctx.grid_step(prob, x0, 0.0, 0.5, 32, False, None, n, st, True)
timeit("unpackbits", lambda: np.unpackbits(pbits.view(np.uint8), axis=1,
                                           bitorder="little")[:, :1000].astype(bool))
print("kernel_ms", res.kernel_ms)
