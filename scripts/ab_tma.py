"""A/B of the two-step rollout's scenario ring at C2: per-lane cp.async (default) vs TMA
bulk copies (tma_ring), event time of L2-flushed steps and the k_grid span, alternated."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi

ctx = _capi.context(0)
stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda", 0))
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
x0 = np.zeros(3)
x0p = x0.ctypes.data
res = _capi.GridResult()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def measure(n=1000):
    ts = []
    with torch.cuda.stream(stream):
        for s in range(420):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sc = _capi.make_scenarios(7 + s, 0, n, m.lo, m.span)
            _capi.check(ctx.lib.rg_grid_step(ctx.handle, prob, x0p, 0.0, 0.5, 32, 0, None, n, 0,
                                             sc, None, None, res,
                                             _capi.RG_ASYNC | _capi.RG_NO_TIMING))
            b.record(stream)
            if s >= 20:
                ts.append((a, b))
            if s % 50 == 49:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
    ev = [x.elapsed_time(y) for x, y in ts]
    spans = []
    for s in range(120):
        sc = _capi.make_scenarios(20000 + s, 0, n, m.lo, m.span)
        _capi.check(ctx.lib.rg_grid_step(ctx.handle, prob, x0p, 0.0, 0.5, 32, 0, None, n, 0, sc,
                                         None, None, res, _capi.RG_NO_TIMING))
        if s >= 20:
            spans.append(res.kernel_ms * 1e3)
    return float(np.median(ev)), float(np.median(spans))


for rep in range(3):
    for tma in (0, 1):
        ctx.set_option("tma_ring", tma)
        e, sp = measure()
        print(f"tma_ring={tma}: event {e:.4f} ms  span {sp:.1f} us", flush=True)
