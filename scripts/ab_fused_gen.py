"""A/B of the fused generator in the single-wave C2 step (rg_set_option "fused_gen"): event
times of 400 L2-flushed steps, three alternations."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
ctx = _capi.context(0)
stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda", 0))
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
x0 = np.zeros(3); x0p = x0.ctypes.data
res = _capi.GridResult()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
def run(opt, steps=400):
    ctx.set_option("fused_gen", 1 - opt)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for s in range(steps + 20):
            flush.zero_()
            if s >= 20: evs[s-20][0].record(stream)
            sc = _capi.make_scenarios(7 + s, 0, 1000, m.lo, m.span)
            _capi.check(ctx.lib.rg_grid_step(ctx.handle, prob, x0p, 0.0, 0.5, 32, 0, None, 1000, 0, sc, None, None, res, _capi.RG_ASYNC | _capi.RG_NO_TIMING))
            if s >= 20: evs[s-20][1].record(stream)
        torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) for a, b in evs])
    out = _capi.GridResult(); _capi.check(ctx.lib.rg_grid_fetch(ctx.handle, None, 32, out))
    assert out.row == 31
    return float(np.mean(t)), float(np.median(t))
for rep in range(3):
    for opt in (1, 0):
        print("no_fused_gen" if opt else "fused_gen   ", run(opt))
