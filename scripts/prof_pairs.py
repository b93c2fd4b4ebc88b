"""ncu driver: the batched step over compacted (episode, row) pairs, C5's closed-loop regime
(one live row per episode: v_prev = r = 0.4), E episodes x 10k scenarios, fused RNG."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2510_08288_b200 as rg  # noqa: E402
from paper_2510_08288_b200 import _capi  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = _capi.context(0)
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
vp = np.full(E, 0.4)
X = np.stack([[np.tanh(v), v, np.tanh(v) / 2] for v in vp])
for s in range(reps):
    out = ctx.grid_step_batch(prob, X, vp, vp, list(range(s * E, (s + 1) * E)), 0, 10_000, m.lo,
                              m.span, 32)
    assert np.all(out[1] == 1.0)
print("ok")
