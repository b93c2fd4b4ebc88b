"""Benchmark of the robust Reference Governor step on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): the bench snapshot of the
reference's bench_sweep (harness.py:269-271) -- surrogate fuel-cell plant,
h = 0.01, Y = [-0.9, 0.9], eps = 0.05, x0 = 0, v_prev = 0, r = 0.5, M = 32
candidates, j* = 256, U(+-0.001) disturbances, 1000 scenarios per GPU, a fresh
scenario seed every step.  All 32 rows are feasible, so one step is exactly
32 * n_sim * 256 cell-steps (one cell-step = one RK4 transition of one
(candidate, scenario) rollout with its fused checks).

  value  device-resident throughput: the fused step kernel (RNG in-kernel, so
         inputs are the step's scalars), CUDA events on the launching stream,
         L2 flushed between steps.  cell-steps/s over all ranks.
  e2e    the same metric through the public API robust_rg_parallel() with
         host buffers in and the KappaResult (incl. P) back on the host.
  --impl reference  the reference's CPU path (oracle C port of the numba
         kernels, kernels.py:47-162, with the reference's fill partition) on
         every host core, same workload.

Multi-GPU (torchrun): rank r takes scenarios [r*n, (r+1)*n) of one global
stream (weak scaling); the per-row violation counts go through one NCCL
all-reduce (MAX) per step and every rank extracts the same row on the device.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "robust RG step latency (ms) at N scenarios; scenario-steps/sec vs FP64 roofline"
UNIT = "cell-steps/s"
FLOPS_PER_CELL_STEP = 210  # 58 explicit ops + 4 tanh x 38
FP64_INSTR_PER_CELL_STEP = 226  # fallback only; bench reads profiles/k_grid_ncu.json (ncu count)
J_STAR, M_GRID, N_PER_GPU, R_REF = 256, 32, 1000, 0.5
BASE_SEED = 7
WORKLOAD = "C2 bench snapshot: robust grid step (Alg. 3)"
CHUNK = 50  # timed steps enqueued per device-side sleep (see run_own)
SLEEP_CYCLES_PER_STEP = 1_000_000  # ~0.5 ms of host enqueue time per step at ~2 GHz


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--n-sim", type=int, default=N_PER_GPU, help="scenarios per GPU")
    ap.add_argument("--j-star", type=int, default=J_STAR)
    ap.add_argument("--e2e-steps", type=int, default=300)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the larger-N points (10k staged, 2^20 fused RNG)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7
                          for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(sm)}


# ---------------------------------------------------------------- CPU baseline

def cpu_baseline(n_sim: int, j_star: int, seconds: float, reps_max: int = 20):
    """The reference's CPU path (oracle port) on this host: multicore on every
    core, plus one serial rep; presampled scenarios like bench_sweep's
    kernel-only mode (harness.py:345-354)."""
    from oracle import oracle as orc

    cores = orc.cpu_count()
    tlo, thi = orc.tighten(-0.9, 0.9, 0.0, 0.05)
    dist = orc.sample(BASE_SEED, n_sim, j_star + 1, [(-0.001, 0.001)] * 3)
    x0 = np.zeros(3)
    cells = M_GRID * n_sim * j_star

    def one(workers):
        t0 = time.perf_counter()
        k, v, feas, _, _, st = orc.grid_step(0.01, x0, 0.0, R_REF, M_GRID, dist, -0.9, 0.9, tlo,
                                             thi, j_star, workers=workers)
        dt = time.perf_counter() - t0
        assert st["early_terms"] == 0 and feas and k == 1.0
        return dt

    one(cores)  # warm-up: thread creation and page faults stay out of the clock
    times, t_end = [], time.perf_counter() + seconds
    while len(times) < reps_max and (not times or time.perf_counter() < t_end):
        times.append(one(cores))
    ser_cells = M_GRID * min(n_sim, 250) * j_star
    d_ser = dist[: min(n_sim, 250)]
    t0 = time.perf_counter()
    orc.grid_step(0.01, x0, 0.0, R_REF, M_GRID, d_ser, -0.9, 0.9, tlo, thi, j_star, workers=1)
    t_ser = time.perf_counter() - t0
    # the same grid step on 8 workers (the survey's host), and the reference's other entry
    # point on the same scenarios: robust_rg_sequential (Alg. 2, one core; at r = 0.5
    # every scenario's kappa = 1 probe is feasible, one rollout per scenario)
    t8 = []
    for _ in range(3):
        t0 = time.perf_counter()
        orc.grid_step(0.01, x0, 0.0, R_REF, M_GRID, dist, -0.9, 0.9, tlo, thi, j_star,
                      workers=min(8, cores))
        t8.append(time.perf_counter() - t0)
    import paper_2510_08288_b200 as rg
    vlo, vhi = rg.admissible_setpoints(tlo, thi)
    t0 = time.perf_counter()
    kap = orc.bisect_all_c(0.01, x0, 0.0, R_REF, -0.9, 0.9, vlo, vhi, dist, j_star, 8)[0]
    t_alg2 = time.perf_counter() - t0
    assert np.all(kap == 1.0)
    best = min(times)
    return {
        "value": cells / best, "unit": UNIT, "cores": cores, "kind": "port",
        "sample": f"{len(times)} robust grid steps (M={M_GRID}, n_sim={n_sim}, j*={j_star}, "
                  f"presampled scenarios) on {cores} threads, best rep",
        "ms_per_step": best * 1e3, "ms_per_step_mean": statistics.mean(times) * 1e3,
        "serial_1core": {"value": ser_cells / t_ser, "unit": UNIT,
                         "sample": f"1 step at n_sim={min(n_sim, 250)}"},
        "multicore_8_workers": {"value": cells / min(t8), "unit": UNIT,
                                "ms_per_step": min(t8) * 1e3, "sample": "best of 3 full steps"},
        "sequential_alg2_1core": {"ms_per_step": t_alg2 * 1e3, "n_sim": n_sim,
                                  "sample": "robust_rg_sequential on the step's scenarios, "
                                            "1 core (C scenario loop)"},
    }


REF_BUDGET_S = 150.0  # the reference arm stops timing after this many seconds of steps


def run_reference(args, rank, world):
    """The reference's CPU path (the oracle's C port of the numba fills, with the
    reference's row/cell partition) on every host core: W untimed steps, then up to
    K timed steps of the full workload (one robust grid step each), stopping early
    once REF_BUDGET_S seconds are spent so the arm ends within a few minutes."""
    if rank != 0:
        return
    from oracle import oracle as orc

    n_sim = args.n_sim * world
    cores = orc.cpu_count()
    tlo, thi = orc.tighten(-0.9, 0.9, 0.0, 0.05)
    x0 = np.zeros(3)
    cells = M_GRID * n_sim * args.j_star

    def one(seed):
        dist = orc.sample(seed, n_sim, args.j_star + 1, [(-0.001, 0.001)] * 3)
        t0 = time.perf_counter()
        k, _, feas, _, _, st = orc.grid_step(0.01, x0, 0.0, R_REF, M_GRID, dist, -0.9, 0.9, tlo,
                                             thi, args.j_star, workers=cores)
        dt = time.perf_counter() - t0
        assert st["early_terms"] == 0 and feas and k == 1.0
        return dt

    for s in range(max(args.warmup, 1)):
        one(BASE_SEED + s)
    times, t_end = [], time.perf_counter() + REF_BUDGET_S
    for s in range(args.steps):
        times.append(one(BASE_SEED + args.warmup + s))
        if time.perf_counter() > t_end:
            break
    total = float(sum(times))
    value = cells * len(times) / total
    cb = {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
          "sample": f"{len(times)} timed robust grid steps of the full workload (M={M_GRID}, "
                    f"n_sim={n_sim}, j*={args.j_star}; scenarios presampled outside the clock) "
                    f"on {cores} threads after {max(args.warmup, 1)} warm-up steps"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": len(times), "steps_requested": args.steps,
        "warmup": args.warmup, "ms_per_step": total * 1e3 / len(times),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_sim": n_sim,
                   "j_star": args.j_star, "m_grid": M_GRID, "plant": "surrogate-fc",
                   "disturbance": "U(+-0.001)", "r": R_REF},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ms_per_step_min": min(times) * 1e3,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- own arm

def run_own(args, rank, world, local_rank):
    import torch

    import paper_2510_08288_b200 as rg
    from paper_2510_08288_b200 import _capi

    # RG_BENCH_DIST_BACKEND=gloo + RG_BENCH_DEVICE=0 smoke-test the N>1 code path on one GPU
    # (the collectives then run on the host; timings of such a run mean nothing)
    backend = os.environ.get("RG_BENCH_DIST_BACKEND", "nccl")
    if "RG_BENCH_DEVICE" in os.environ:
        local_rank = int(os.environ["RG_BENCH_DEVICE"])
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    ctx = _capi.context(local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda", local_rank))

    n_sim, j_star = args.n_sim, args.j_star
    k0 = rank * n_sim
    cells_rank = M_GRID * n_sim * j_star
    plant = rg.make_plant("surrogate-fc")
    box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
    tight = rg.tighten(box, 0.05)
    v_lo, v_hi = rg.admissible_setpoints(tight.lower, tight.upper)
    prob = _capi.Problem(0.01, -0.9, 0.9, v_lo, v_hi, j_star, 0)
    model = rg.DisturbanceModel.scaled(0.001, 3)
    x0 = np.zeros(3)
    lib = ctx.lib
    res = _capi.GridResult()
    viol = torch.zeros(M_GRID, dtype=torch.int32, device=f"cuda:{local_rank}")
    flags = _capi.RG_ASYNC | _capi.RG_NO_TIMING
    if world > 1:
        flags |= _capi.RG_DEVICE_PTRS
    x0_ptr = x0.ctypes.data_as(ctypes_vp())  # kernel parameter: host memory
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32,
                        device=f"cuda:{local_rank}")
    row_idx = torch.arange(M_GRID, dtype=torch.int32, device=f"cuda:{local_rank}")
    minus1 = torch.full_like(row_idx, -1)

    def step(s):
        scen = _capi.make_scenarios(BASE_SEED + s, k0, n_sim, model.lo, model.span)
        _capi.check(lib.rg_grid_step(ctx.handle, prob, x0_ptr, 0.0, R_REF, M_GRID, 0, None,
                                     n_sim, 0, scen,
                                     ctypes_vp()(viol.data_ptr()) if world > 1 else None,
                                     None, res, flags))
        if world > 1:
            # per-row violating-scenario counts, int32 (a gated-out row is -1 on every
            # rank): the global MAX is 0 exactly for the rows feasible on every shard
            torch.distributed.all_reduce(viol, op=torch.distributed.ReduceOp.MAX)
            return torch.where(viol == 0, row_idx, minus1).max()  # literal Eq. 4
        return None

    with torch.cuda.stream(stream):
        for s in range(args.warmup):
            step(s)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        sampler = ClockSampler(local_rank)
        sampler.start()
        time.sleep(0.2)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        # The timed steps are enqueued in chunks behind a device-side sleep, so
        # the device never idles waiting for the host to submit the next step
        # inside an event pair (the host needs ~0.2 ms per step to enqueue a
        # flush, two events and the step; the device ~0.22 ms to run them).
        wall = 0.0
        for c0 in range(0, args.steps, CHUNK):
            c1 = min(args.steps, c0 + CHUNK)
            torch.cuda._sleep(int(SLEEP_CYCLES_PER_STEP * (c1 - c0)))
            w0 = time.perf_counter()
            for s in range(c0, c1):
                flush.zero_()  # L2 (126 MB) flush between timed steps, outside the events
                ev[s][0].record(stream)
                step(args.warmup + s)
                ev[s][1].record(stream)
            torch.cuda.synchronize()
            wall += time.perf_counter() - w0
        if world > 1:
            torch.distributed.barrier()
        clocks = sampler.stop()
    per = np.array([a.elapsed_time(b) for a, b in ev])  # ms
    total_ms = float(per.sum())
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{local_rank}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    # the step's decision must be the reference's: all 32 rows feasible -> kappa = 1
    out = _capi.GridResult()
    _capi.check(lib.rg_grid_fetch(ctx.handle, None, M_GRID, out))
    if world == 1:
        assert out.row == M_GRID - 1 and out.early_terms == 0, (out.row, out.early_terms)

    # k_gen_soa + k_grid when the scenario block is staged in L2, k_grid alone when fused
    launches_per_step = 2 if n_sim * j_star * 24 <= (16 << 30) else 1
    cells_total = cells_rank * world * args.steps
    value = cells_total / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps

    # dominant kernel: k_grid.  The event pair brackets the step (k_gen_soa +
    # k_grid when staged); the ncu launch list (profiles/) gives k_grid's share.
    kernel_ms = float(np.mean(per)) if world == 1 else None
    peak = ctx.fp64_peak()
    roof = None
    if kernel_ms:
        achieved = FLOPS_PER_CELL_STEP * cells_rank / (kernel_ms * 1e-3)
        # the instruction-mix view: FP64-pipe instructions per cell-step as
        # counted by ncu on this kernel (profiles/k_grid_ncu.json); the 210-flop
        # convention counts each division as 1 flop
        fp64_per_cell = _ncu_summary().get("fp64_instr_per_cell_step", FP64_INSTR_PER_CELL_STEP)
        fp64_instr_rate = cells_rank / (kernel_ms * 1e-3) * fp64_per_cell
        roof = {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": _ncu_traffic(),
                "fp64_pipe_frac": fp64_instr_rate / (peak / 2.0),
                "issue_model": issue_model(n_sim, j_star, kernel_ms, clocks),
                "fp64_instr_per_cell_step": fp64_per_cell,
                "peak_source": "measured in this run: rg_fp64_peak (independent DFMA chains, "
                               "2 flop per DFMA); MEASURED_PEAKS.json has no FP64 figure",
                "flops_per_cell_step": FLOPS_PER_CELL_STEP, "cell_steps_per_launch": cells_rank,
                "kernel_ms": kernel_ms}

    # e2e through the public API with host buffers (rank-local shard)
    e2e = None
    if world == 1:
        cfg = rg.GovernorConfig(j_star=j_star, m_grid=M_GRID, n_sim=n_sim)
        for s in range(5):
            rg.robust_rg_parallel(plant, x0, rg.GovernorState(0.0), R_REF, box,
                                  rg.sample_scenarios(model, n_sim, j_star + 1, seed=s), cfg)
        t0 = time.perf_counter()
        for s in range(args.e2e_steps):
            scen = rg.sample_scenarios(model, n_sim, j_star + 1, seed=BASE_SEED + s)
            r = rg.robust_rg_parallel(plant, x0, rg.GovernorState(0.0), R_REF, box, scen, cfg)
        t_e2e = (time.perf_counter() - t0) / args.e2e_steps
        assert r.kappa_opt == 1.0 and r.matrix.all()
        h2d = 3 * 8 + 2 * 8 + 9 * 8   # x0, v_prev/r, scenario stream descriptor (kernel params)
        d2h = (M_GRID * ((n_sim + 31) // 32) * 4) + M_GRID * 4 + 64  # P bits, counts, result
        e2e = {"value": cells_rank / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e * 1e3,
               "api": "paper_2510_08288_b200.robust_rg_parallel (keep_matrix=True)"}

    # latency split of one synchronous step (the C ABI call a user makes, no P):
    # host call -> result in host memory, the device span of k_grid (first block
    # start to publication, globaltimer), and the final reduction inside it
    latency = None
    if world == 1:
        sync_res = _capi.GridResult()
        walls, spans, reds = [], [], []
        for s in range(220):
            scen = _capi.make_scenarios(BASE_SEED + 20000 + s, k0, n_sim, model.lo, model.span)
            t0 = time.perf_counter()
            _capi.check(lib.rg_grid_step(ctx.handle, prob, x0_ptr, 0.0, R_REF, M_GRID, 0, None,
                                         n_sim, 0, scen, None, None, sync_res,
                                         _capi.RG_NO_TIMING))
            dt = time.perf_counter() - t0
            if s >= 20:
                walls.append(dt * 1e6)
                spans.append(sync_res.kernel_ms * 1e3)
                reds.append(sync_res.reduce_us)
        latency = {"api_call_us": float(np.median(walls)),
                   "k_grid_span_us": float(np.median(spans)),
                   "launch_overhead_us": float(np.median(walls) - np.median(spans)),
                   "reduction_us": float(np.median(reds)),
                   "note": "median of 200 synchronous rg_grid_step calls at the workload "
                           "(no P): api_call = host wall time of the call; k_grid_span = "
                           "first block start to result publication (device globaltimer); "
                           "launch_overhead = the difference (host enqueue, launch latency, "
                           "k_gen_soa, result visibility); reduction = the last block's row "
                           "extraction and publication inside the span"}

    # larger scenario counts (BASELINE C3 size and the C4 shard size), same step
    sweep = []
    if world == 1 and not args.no_sweep:
        for n_big, reps in ((10_000, 20), (1 << 20, 3)):
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(reps + 1)]
            with torch.cuda.stream(stream):
                for s_i, (a, b) in enumerate(evs):
                    flush.zero_()
                    a.record(stream)
                    sc = _capi.make_scenarios(BASE_SEED + 1000 + s_i, 0, n_big, model.lo,
                                              model.span)
                    _capi.check(lib.rg_grid_step(ctx.handle, prob, x0_ptr, 0.0, R_REF, M_GRID, 0,
                                                 None, n_big, 0, sc, None, None, res, flags))
                    b.record(stream)
                torch.cuda.synchronize()
            t = np.array([a.elapsed_time(b) for a, b in evs[1:]])
            cells = M_GRID * n_big * j_star
            rate = cells / (t.mean() * 1e-3)
            sweep.append({"n_sim": n_big, "ms_per_step": float(t.mean()), "value": rate,
                          "unit": UNIT, "roofline_frac": FLOPS_PER_CELL_STEP * rate / peak,
                          "issue_frac": issue_model(n_big, j_star, float(t.mean()),
                                                    clocks)["frac"],
                          "rng": "staged" if n_big * j_star * 24 <= (16 << 30) else "fused"})

    if world > 1:
        from paper_2510_08288_b200.sharded import robust_rg_parallel_sharded
        cfg = rg.GovernorConfig(j_star=j_star, m_grid=M_GRID, n_sim=n_sim * world,
                                device=local_rank)
        for s in range(3):
            robust_rg_parallel_sharded(plant, x0, rg.GovernorState(0.0), R_REF, box,
                                       rg.sample_scenarios(model, n_sim * world, j_star + 1,
                                                           seed=s, device=local_rank), cfg)
        torch.distributed.barrier()
        t0 = time.perf_counter()
        for s in range(args.e2e_steps):
            scen = rg.sample_scenarios(model, n_sim * world, j_star + 1, seed=BASE_SEED + s,
                                       device=local_rank)
            r = robust_rg_parallel_sharded(plant, x0, rg.GovernorState(0.0), R_REF, box, scen,
                                           cfg)
        t = torch.tensor([(time.perf_counter() - t0) / args.e2e_steps], dtype=torch.float64,
                         device=f"cuda:{local_rank}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(t.item())
        assert r.kappa_opt == 1.0
        e2e = {"value": cells_rank * world / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": 112, "d2h_bytes_per_step": M_GRID * 4 + 64,
               "ms_per_step": t_e2e * 1e3,
               "api": "paper_2510_08288_b200.sharded.robust_rg_parallel_sharded"}

    # C5 shape: a batch of independent episodes in one launch (64 x 10k scenarios,
    # bench snapshot so every row runs the full horizon), and C3: the desk-scale
    # closed loop at 10k scenarios (the whole 2000-step trace)
    if world == 1 and not args.no_sweep:
        E, n_b = 64, 10_000
        cfg_b = rg.GovernorConfig(j_star=j_star, m_grid=M_GRID, n_sim=n_b)
        seeds = [BASE_SEED + 5000 + e for e in range(E)]
        rg.robust_rg_parallel_batch(plant, np.zeros((E, 3)), np.zeros(E), np.full(E, R_REF),
                                    box, model, n_b, seeds, cfg_b)
        t0 = time.perf_counter()
        kap_b, _, _, _ = rg.robust_rg_parallel_batch(plant, np.zeros((E, 3)), np.zeros(E),
                                                     np.full(E, R_REF), box, model, n_b, seeds,
                                                     cfg_b)
        t_b = time.perf_counter() - t0
        assert np.all(kap_b == 1.0)
        sweep.append({"workload": f"C5 shape: batch of {E} episodes x {n_b} scenarios, one launch",
                      "ms_per_step": t_b * 1e3, "value": E * M_GRID * n_b * j_star / t_b,
                      "unit": UNIT, "timing": "wall clock around the synchronous API call"})
        from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop
        prof = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
        t0 = time.perf_counter()
        rec = run_closed_loop(plant, box, model, rg.GovernorConfig(n_sim=10_000), prof, 2000, 2024)
        t_c3 = time.perf_counter() - t0
        sweep.append({"workload": "C3: desk-scale closed loop, n_sim=10000, the full 2000-step trace",
                      "ms_per_step": t_c3 * 1e3 / 2000, "violations": rec.violations(box),
                      "timing": "wall clock, host true-plant step included (reference: "
                                "~650 ms/step on 8 CPU cores, SURVEY.md §6)"})
        # the bisection searches on a transient step (r=2.5 from rest, kappa* = 0.5078):
        # exact Alg. 2 (per-scenario bisections, min) and the joint search (one kappa
        # for all scenarios per iteration, OR-reduced flag); both land on the same kappa
        # Alg. 2 on the C2 step itself (r = 0.5: one feasible rollout per scenario), the
        # device side of cpu_baseline.sequential_alg2_1core
        sc = _capi.make_scenarios(BASE_SEED, k0, n_sim, model.lo, model.span)
        ctx.bisect(prob, x0, 0.0, R_REF, 8, None, n_sim, sc)
        t0 = time.perf_counter()
        for _ in range(20):
            res_b = ctx.bisect(prob, x0, 0.0, R_REF, 8, None, n_sim, sc)[0]
        sweep.append({"workload": f"bisection (alg2), C2 snapshot r=0.5, n_sim={n_sim}",
                      "ms_per_step": (time.perf_counter() - t0) / 20 * 1e3,
                      "kappa": float(res_b.kappa), "rollouts": int(res_b.cells),
                      "timing": "wall clock around the synchronous C-ABI call"})
        for n_b in (10_000, 1 << 20):
            sc = _capi.make_scenarios(BASE_SEED + 9000, 0, n_b, model.lo, model.span)
            for name, call in (
                    ("alg2", lambda: ctx.bisect(prob, x0, 0.0, 2.5, 8, None, n_b, sc)[0]),
                    ("joint", lambda: ctx.bisect_joint(prob, x0, 0.0, 2.5, 8, None, n_b, sc))):
                call()
                reps = 10
                t0 = time.perf_counter()
                for _ in range(reps):
                    res_b = call()
                t_b = (time.perf_counter() - t0) / reps
                sweep.append({"workload": f"bisection ({name}), r=2.5 transient, n_sim={n_b}",
                              "ms_per_step": t_b * 1e3, "kappa": float(res_b.kappa),
                              "rollouts": int(res_b.cells),
                              "timing": "wall clock around the synchronous C-ABI call"})

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c = cpu_baseline(n_sim, j_star, args.cpu_seconds)
        cb = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}
        for k in ("serial_1core", "multicore_8_workers", "sequential_alg2_1core"):
            cb[k] = c[k]

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD,
                       "rng": ("staged (k_gen_soa + k_grid)" if launches_per_step == 2
                               else "fused (k_grid)"),
                       "n_sim": n_sim * world, "n_sim_per_gpu": n_sim, "j_star": j_star,
                       "m_grid": M_GRID, "plant": "surrogate-fc", "disturbance": "U(+-0.001)",
                       "r": R_REF, "cell_steps_per_step": cells_rank * world,
                       "l2": "flushed between timed steps (256 MB write, outside the events)",
                       "parallelism": f"scenario shards x{world}" + (", NCCL all-reduce of "
                                                                     "row counts (MAX)" if world > 1
                                                                     else "")},
            "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "latency": latency,
            "sweep": sweep,
            "gpu_launches": args.steps * launches_per_step, "clocks": clocks,
            "host_enqueue_ms_per_step": wall * 1e3 / args.steps,  # incl. the chunks' device sleep
            "kernel_ms_p50": float(np.median(per)), "kernel_ms_min": float(per.min()),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def ctypes_vp():
    import ctypes
    return ctypes.c_void_p


def _ncu_summary(name="k_grid_ncu.json"):
    """A committed ncu --set full summary of k_grid (scripts/ncu_summary.py): at C2
    by default, k_grid_ncu_10k.json for the multi-wave form."""
    p = ROOT / "profiles" / name
    try:
        return json.loads(p.read_text())
    except (OSError, ValueError):
        return {}


def issue_model(n_sim, j_star, ms, clocks, sm_count=148):
    """The rollout's instruction-issue bound.  Each SM sub-partition (SMSP) issues
    one warp-instruction per cycle, and an FP64 warp-instruction holds the issue
    slot for two (16 FP64 lanes per SMSP): a warp-step costs 2*FP64 + other cycles
    (ncu counts, profiles/k_grid_ncu.json).  Bound = all warp-steps spread evenly
    over the 4*148 SMSPs at the measured SM clock; frac = bound / measured."""
    # the single-wave step runs the integer tanh forms (profiles/k_grid_ncu.json, C2),
    # above one wave the operand-modifier forms (profiles/k_grid_ncu_10k.json)
    single_wave = (n_sim + 255) // 256 * M_GRID <= sm_count
    ncu = _ncu_summary() if single_wave else _ncu_summary("k_grid_ncu_10k.json")
    fp64 = ncu.get("fp64_instr_per_cell_step")
    total = ncu.get("instr_per_cell_step")
    if not fp64 or not total or not ms:
        return {"frac": None}
    cyc = 2.0 * fp64 + (total - fp64)
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    warp_steps = (n_sim + 31) // 32 * M_GRID * j_star
    bound_ms = warp_steps / (4 * sm_count) * cyc / (mhz * 1e3)
    return {"cycles_per_warp_step": cyc, "bound_ms": bound_ms, "frac": bound_ms / ms,
            "instr_source": ncu.get("workload"),
            "note": "2 issue cycles per FP64 warp-instruction + 1 per other, all warp-steps "
                    "balanced over 592 SMSPs (at 1000 scenarios the 1000 warps cannot "
                    "balance below 2 per loaded SMSP: that bound is 1.16x this one)"}


def _ncu_traffic():
    """dram bytes per k_grid launch from the committed ncu --set full summary."""
    return _ncu_summary().get("dram_bytes_per_launch")


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_own(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
