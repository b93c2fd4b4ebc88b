"""Grid step device time with the scenario block staged (k_gen_soa + SoA reads) versus
fused (counter RNG in the rollout), at several scenario counts."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2510_08288_b200 as rg  # noqa: E402
from paper_2510_08288_b200 import _capi  # noqa: E402

ctx = _capi.context(0)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
import torch  # noqa: E402

st = torch.cuda.ExternalStream(ctx.stream_ptr)
for n in [int(a) for a in sys.argv[1:]]:
    row = [f"N={n:8d}"]
    for mode in ("staged", "fused"):
        ts = []
        for s in range(6):
            sc = _capi.make_scenarios(7 + s, 0, n, m.lo, m.span)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            res, _, _ = ctx.grid_step(prob, np.zeros(3), 0.0, 0.5, 32, False, None, n, sc, False,
                                      rng_mode=mode, timing=False)
            b.record(st)
            b.synchronize()
            if s:
                ts.append(a.elapsed_time(b))
        row.append(f"{mode} {np.median(ts):9.3f} ms ({32 * n * 256 / np.median(ts) / 1e6:.1f} G/s)")
    print("  ".join(row), flush=True)
