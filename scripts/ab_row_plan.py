"""A/B of the host row plan and the single-wave rollout form on closed-loop-like steps: one
live row (v_prev = r) and a transient (v_prev != r, gated rows) at 1k-30k scenarios, event
times of L2-flushed steps; then the C3 closed loop under each setting."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi
from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop
ctx = _capi.context(0)
stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda", 0))
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
res = _capi.GridResult()
SETS = {"plan+ts": dict(no_row_plan=0, no_step2=0, no_ts=0, ts_staged=0),
        "plan+ts staged": dict(no_row_plan=0, no_step2=0, no_ts=0, ts_staged=1),
        "plan+s2 (no ts)": dict(no_row_plan=0, no_step2=0, no_ts=1),
        "device rows": dict(no_row_plan=1, no_step2=0, no_ts=1, ts_staged=0)}
if len(sys.argv) > 1 and sys.argv[1] == "ts":  # the time-split A/B only, twice
    SETS = {"plan+ts": SETS["plan+ts"], "plan+ts staged": SETS["plan+ts staged"],
            "plan+s2 (no ts)": SETS["plan+s2 (no ts)"], "plan+ts again": SETS["plan+ts"],
            "plan+ts staged again": SETS["plan+ts staged"]}


def step_time(n, vp, r, reps=30):
    x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]); x0p = x0.ctypes.data
    ts = []
    with torch.cuda.stream(stream):
        for s in range(reps + 1):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sc = _capi.make_scenarios(7 + s, 0, n, m.lo, m.span)
            _capi.check(ctx.lib.rg_grid_step(ctx.handle, prob, x0p, vp, r, 32, 0, None, n, 0, sc,
                                             None, None, res, _capi.RG_ASYNC | _capi.RG_NO_TIMING))
            b.record(stream)
            torch.cuda.synchronize()
            if s:
                ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for name, opts in SETS.items():
    for k, v in opts.items():
        ctx.set_option(k, v)
    line = [name]
    for n in (1000, 10_000, 30_000):
        line.append(f"n={n}: 1-row {step_time(n, 0.4, 0.4):.4f} transient {step_time(n, 1.2, 2.5):.4f}")
    prof = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
    t0 = time.perf_counter()
    run_closed_loop(rg.make_plant("surrogate-fc"), rg.ConstraintSet(-0.9, 0.9, 0.0), m,
                    rg.GovernorConfig(n_sim=10_000), prof, 2000, 2024)
    line.append(f"C3 {(time.perf_counter() - t0) / 2000 * 1e3:.4f} ms/step")
    print(" | ".join(line), flush=True)
