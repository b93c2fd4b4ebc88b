"""Host-side cost of one C2 grid step through the C ABI, piece by piece."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_08288_b200 as rg  # noqa: E402
from paper_2510_08288_b200 import _capi, governor as G  # noqa: E402

ctx = _capi.context(0)
lib = ctx.lib
N = 400


def timeit(name, fn):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    dt = (time.perf_counter() - t0) / N * 1e6
    print(f"{name:50s} {dt:8.1f} us")
    return dt


timeit("ctypes no-op (rg_abi_version)", lambda: lib.rg_abi_version())
prob, iv, grid, grid_list = G._prepared(0.01, -0.9, 0.9, 0.0, 0.05, "scale", 256, 32)
model = rg.DisturbanceModel.scaled(0.001, 3)
sc = _capi.make_scenarios(7, 0, 1000, model.lo, model.span)
x0 = np.zeros(3)
for mode in (None, "fused", "staged"):
    timeit(f"ctx.grid_step rng={mode} no pbits", lambda: ctx.grid_step(
        prob, x0, 0.0, 0.5, 32, False, None, 1000, sc, False, rng_mode=mode))
res = _capi.GridResult()
x0p = x0.ctypes.data_as(ctypes.c_void_p)
for flags, name in ((0, "default"), (_capi.RG_NO_TIMING, "no timing"),
                    (_capi.RG_NO_TIMING | _capi.RG_FUSED_RNG, "no timing, fused")):
    timeit(f"raw rg_grid_step {name}", lambda: _capi.check(lib.rg_grid_step(
        ctx.handle, ctypes.byref(prob), x0p, 0.0, 0.5, 32, 0, None, 1000, 0, ctypes.byref(sc),
        None, None, ctypes.byref(res), flags)))
# device-side span of one call (first kernel start .. D2H end) via events on the lib stream
stream = torch.cuda.ExternalStream(ctx.stream_ptr()) if hasattr(ctx, "stream_ptr") else None
if stream is not None:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    spans = []
    for _ in range(50):
        a.record(stream)
        _capi.check(lib.rg_grid_step(ctx.handle, ctypes.byref(prob), x0p, 0.0, 0.5, 32, 0, None,
                                     1000, 0, ctypes.byref(sc), None, None, ctypes.byref(res),
                                     _capi.RG_NO_TIMING))
        b.record(stream)
        b.synchronize()
        spans.append(a.elapsed_time(b) * 1e3)
    print(f"{'device span of one call (events around it)':50s} {np.median(spans):8.1f} us")
print("kernel_us (events inside, k_grid only)", res.kernel_ms * 1e3)
