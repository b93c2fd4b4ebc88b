"""Distribution of per-step device times of the C2 grid step under bench.py's loop,
with and without the nvidia-smi clock sampler and the L2 flush (outlier hunt).

usage: python scripts/timing_dist.py [steps]
"""
import ctypes
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_08288_b200 as rg  # noqa: E402
from paper_2510_08288_b200 import _capi  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
ctx = _capi.context(0)
stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda", 0))
tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9), 0.05)
lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
prob = _capi.Problem(0.01, -0.9, 0.9, lo, hi, 256, 0)
m = rg.DisturbanceModel.scaled(0.001, 3)
x0 = np.zeros(3)
res = _capi.GridResult()
flags = _capi.RG_ASYNC | _capi.RG_NO_TIMING
x0p = x0.ctypes.data_as(ctypes.c_void_p)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")


def step(seed):
    sc = _capi.make_scenarios(seed, 0, 1000, m.lo, m.span)
    _capi.check(ctx.lib.rg_grid_step(ctx.handle, prob, x0p, 0.0, 0.5, 32, 0, None, 1000, 0, sc,
                                     None, None, res, flags))


def run(tag, do_flush, sampler, chunk):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    smi = None
    if sampler:
        smi = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm",
                                "--format=csv,noheader", "-lms", "50"],
                               stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    with torch.cuda.stream(stream):
        for s in range(20):
            step(7 + s)
        torch.cuda.synchronize()
        for c0 in range(0, steps, chunk):
            c1 = min(steps, c0 + chunk)
            torch.cuda._sleep(1_000_000 * (c1 - c0))
            for s in range(c0, c1):
                if do_flush:
                    flush.zero_()
                ev[s][0].record(stream)
                step(100 + s)
                ev[s][1].record(stream)
            torch.cuda.synchronize()
    if smi:
        smi.terminate()
        smi.wait()
    t = np.array([a.elapsed_time(b) for a, b in ev]) * 1e3  # us
    p = np.percentile(t, [1, 10, 50, 90, 99])
    big = np.nonzero(t > 1.15 * p[2])[0]
    print(f"{tag:34s} mean {t.mean():7.1f} p1 {p[0]:6.1f} p10 {p[1]:6.1f} p50 {p[2]:6.1f} "
          f"p90 {p[3]:6.1f} p99 {p[4]:6.1f} max {t.max():7.1f} us; >1.15*p50: {len(big)} "
          f"(first positions mod chunk: {(big % chunk)[:12].tolist()})", flush=True)


import os  # noqa: E402
tpb = os.environ.get("RG_FORCE_TPB", "auto")
run(f"tpb {tpb}: flush, chunk 50", True, False, 50)
run(f"tpb {tpb}: no flush, chunk 50", False, False, 50)
