"""Benchmark of the robust Reference Governor step on B200 (one JSON line on rank 0).

Workloads (BASELINE.json configs; metric "robust RG step latency (ms) at N scenarios;
scenario-steps/sec vs FP64 roofline", unit cell-steps/s):

  c2  (configs[1], the default at N=1)  the bench snapshot of the reference's
      bench_sweep (harness.py:269-271): surrogate fuel-cell plant, h = 0.01,
      Y = [-0.9, 0.9], eps = 0.05, x0 = 0, v_prev = 0, r = 0.5, M = 32 candidates,
      j* = 256, U(+-0.001) disturbances, 1000 scenarios per GPU, a fresh scenario
      seed every step.  All 32 rows are feasible, so one step is exactly
      32 * n_sim * 256 cell-steps.
  c4  (configs[3], the default at N>1)  the same step over 2^20 scenarios, sharded
      over the N GPUs (strong scaling): rank r simulates the counter range
      [r*n/N, (r+1)*n/N) of one stream (no scenario traffic); the per-row violation
      counts go through one all-reduce (MAX, int32) per step and every rank extracts
      the same row on its device.
  c1  (configs[0])  the desk-scale closed loop with the nominal bisection governor
      (bisection_rg, one scenario, n_kappa 8), the whole 2000-step trace, as one device
      kernel (rg_closed_loop_bisection); the reference arm runs the reference's own loop.
  c3  (configs[2])  the desk-scale closed loop at 10k scenarios per step, the whole
      2000-step setpoint trace (seed 2024): the whole loop as one device kernel
      (rg_closed_loop: governor, kappa, v_t and the true plant on the device);
      at N>1 every rank runs its own episode (seed 2024 + rank, replicas).
  c5  (configs[4])  4096 independent desk-scale closed-loop episodes x 10k scenarios
      (episode seeds 2024 + e), episodes spread over the N GPUs as replicas; K timed
      closed-loop steps after W warm-up steps of the trace.

  value  device-resident throughput, CUDA events on the launching stream, L2 flushed
         between timed steps, max over ranks.
  e2e    the same metric through the public API (robust_rg_parallel, or its sharded
         form at N>1) with host inputs and the result back on the host.
  --impl reference  the reference's own CPU path on the host cores: the unmodified
         refgov package (numba, backend "multicore") staged by oracle/Makefile into
         oracle/_ref, on the same workload (a bounded sample of it per step for c4/c5);
         the oracle's C port of the numba fills when the reference cannot import.

`python bench.py --gpus N` with N > 1 launches N ranks itself (torch.distributed.run)
unless it already runs under torchrun, in which case N must equal WORLD_SIZE.
RG_BENCH_DIST_BACKEND=gloo + RG_BENCH_DEVICE=0 run the N>1 code path on one GPU (the
collectives then run through gloo; the timings of such a run mean nothing).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# The multi-rank code path (torch.distributed, the per-step all-reduce) runs when
# WORLD_SIZE > 1, or at world size 1 with RG_BENCH_FORCE_DIST=1 (NCCL with one rank: the
# N>1 path exercised end to end on a one-GPU box).  Set in main().
MULTI = False

METRIC = "robust RG step latency (ms) at N scenarios; scenario-steps/sec vs FP64 roofline"
UNIT = "cell-steps/s"
FLOPS_PER_CELL_STEP = 210  # 58 explicit ops + 4 tanh x 38
FP64_INSTR_PER_CELL_STEP = 226  # fallback only; bench reads profiles/k_grid_ncu.json (ncu count)
J_STAR, M_GRID, R_REF = 256, 32, 0.5
BASE_SEED = 7
CHUNK = 50  # timed steps enqueued per device-side sleep (see run_grid)
SLEEP_CYCLES_PER_STEP = 1_000_000  # ~0.5 ms of host enqueue time per step at ~2 GHz
L2_NOTE = "device arm: L2 (126 MB) flushed between timed steps by a 256 MB write outside the events"

WORKLOADS = {
    "c2": {"name": "C2 bench snapshot: robust grid step (Alg. 3), 1000 scenarios per GPU",
           "n_per_gpu": 1000, "scaling": "weak", "steps": 3000, "warmup": 20},
    "c4": {"name": "C4: robust grid step (Alg. 3) over 2^20 scenarios sharded across the GPUs",
           "n_total": 1 << 20, "scaling": "strong", "steps": 20, "warmup": 3},
    "c1": {"name": "C1: desk-scale closed loop with the nominal bisection governor "
                   "(bisection_rg, one scenario), the whole 2000-step trace",
           "n_sim": 1, "scaling": "weak", "steps": 2000, "warmup": 200},
    "c3": {"name": "C3: desk-scale closed loop, 10k scenarios per step, the whole 2000-step trace",
           "n_sim": 10_000, "scaling": "weak", "steps": 2000, "warmup": 200},
    "c5": {"name": "C5: 4096 desk-scale closed-loop episodes x 10k scenarios, episodes as "
                   "replicas across the GPUs", "episodes": 4096, "n_sim": 10_000,
           "scaling": "strong", "steps": 5, "warmup": 3},
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--n-sim", type=int, default=None,
                    help="c2: scenarios per GPU; c4: total scenarios; c5: scenarios per episode")
    ap.add_argument("--episodes", type=int, default=None, help="c5: total episodes")
    ap.add_argument("--j-star", type=int, default=J_STAR)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--xchg", default="nccl", choices=["nccl", "p2p"],
                    help="N>1 grid steps: the row counts' all-reduce through NCCL, or fused into "
                         "the step kernel over NVLink (rg_xchg_*, RG_XCHG)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the extra sizes and entry points (10k, 2^20, C5 shape, C3, "
                         "bisections, dense-input e2e)")
    args = ap.parse_args()
    return args


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


def resolve(args, world):
    wl = args.workload if args.workload != "auto" else ("c2" if world == 1 else "c4")
    spec = dict(WORKLOADS[wl])
    args.steps = spec["steps"] if args.steps is None else args.steps
    args.warmup = spec["warmup"] if args.warmup is None else args.warmup
    if args.e2e_steps is None:
        args.e2e_steps = {"c1": 0, "c2": 300, "c3": 0, "c4": 5, "c5": 0}[wl]
    if wl == "c2":
        spec["n_per_gpu"] = args.n_sim or spec["n_per_gpu"]
    elif wl == "c4":
        spec["n_total"] = args.n_sim or spec["n_total"]
    elif wl == "c3":
        spec["n_sim"] = args.n_sim or spec["n_sim"]
    elif wl == "c1":
        pass
    else:
        spec["n_sim"] = args.n_sim or spec["n_sim"]
        spec["episodes"] = args.episodes or spec["episodes"]
    return wl, spec


def config_of(wl, spec, world, j_star):
    """The workload's config dict -- identical in both arms (same_config)."""
    base = {"plant": "surrogate-fc", "j_star": j_star, "m_grid": M_GRID, "l2": L2_NOTE}
    if wl == "c2":
        return {"workload": spec["name"], "n_sim": spec["n_per_gpu"] * world,
                "disturbance": "U(+-0.001)", "r": R_REF, **base}
    if wl == "c4":
        return {"workload": spec["name"], "n_sim": spec["n_total"], "disturbance": "U(+-0.001)",
                "r": R_REF, **base}
    if wl == "c1":
        return {"workload": spec["name"], "n_sim": 1, "n_kappa": 8,
                "disturbance": "none in the prediction; the true plant's U(+-0.001) (desk-scale "
                "preset)", "profile": "desk-scale [[0,0.4],[400,2.5],[1000,-2.5],[1600,0.2]]",
                "seed": "2024 (+ rank at N>1)", "plant": "surrogate-fc", "j_star": j_star,
                "l2": L2_NOTE}
    if wl == "c3":
        return {"workload": spec["name"], "n_sim": spec["n_sim"],
                "disturbance": "U(+-0.001) (desk-scale preset)", "profile": "desk-scale "
                "[[0,0.4],[400,2.5],[1000,-2.5],[1600,0.2]]", "seed": "2024 (+ rank at N>1)",
                **base}
    return {"workload": spec["name"], "episodes": spec["episodes"], "n_sim": spec["n_sim"],
            "disturbance": "U(+-0.001) (desk-scale preset)", "profile": "desk-scale "
            "[[0,0.4],[400,2.5],[1000,-2.5],[1600,0.2]]", "seeds": "2024 + e", **base}


def self_launch(args):
    """`bench.py --gpus N` outside torchrun: run N ranks through torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), str(ROOT / "bench.py")] + sys.argv[1:]
    return subprocess.call(cmd)


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


# ---------------------------------------------------------------- CPU side (reference)

class RefCPU:
    """The reference's CPU path on this host: the unmodified refgov package (oracle/_ref,
    numba, backend "multicore" = every core) when it imports, else the oracle's C port of
    the numba fills (oracle/rg_oracle.c) on every core.  Test infrastructure only: this is
    the timed baseline, never the product."""

    def __init__(self):
        from oracle import reference

        self.ref, why = reference.load()
        self.kind = "reference" if self.ref is not None else "port"
        self.why_port = why
        if self.ref is not None:
            self.threads = reference.threads
        else:
            from oracle import oracle as orc
            self.orc = orc

    def cores(self):
        if self.ref is not None:
            return self.threads()["numba_num_threads"]
        return self.orc.cpu_count()

    def info(self):
        if self.ref is not None:
            return {"impl": "refgov (unmodified, oracle/_ref) robust_rg_parallel backend="
                            "'multicore', workers=None", **self.threads()}
        return {"impl": "oracle C port of the numba fills (rg_oracle.c)", "why": self.why_port}

    # -- grid step (robust_rg_parallel) on n scenarios of the bench snapshot
    def scenarios(self, n, j_star, seed):
        if self.ref is not None:
            m = self.ref.DisturbanceModel.scaled(0.001, 3)
            return self.ref.sample_scenarios(m, n, j_star + 1, seed=seed)
        return self.orc.sample(seed, n, j_star + 1, [(-0.001, 0.001)] * 3)

    def grid_step(self, scen, n, j_star, workers=None):
        """One robust grid step at the snapshot; returns seconds.  Asserts the reference's
        decision (all rows feasible, kappa = 1)."""
        if self.ref is not None:
            rf = self.ref
            cfg = rf.GovernorConfig(j_star=j_star, m_grid=M_GRID, n_sim=n,
                                    backend="multicore" if workers != 1 else "serial",
                                    workers=workers)
            box = rf.ConstraintSet(-0.9, 0.9, anchor=0.0)
            plant = rf.make_plant("surrogate-fc")
            t0 = time.perf_counter()
            res = rf.robust_rg_parallel(plant, np.zeros(3), rf.GovernorState(0.0), R_REF, box,
                                        scen, cfg)
            dt = time.perf_counter() - t0
            assert res.kappa_opt == 1.0 and res.diagnostics["early_terms"] == 0
            return dt
        orc = self.orc
        tlo, thi = orc.tighten(-0.9, 0.9, 0.0, 0.05)
        t0 = time.perf_counter()
        k, _, feas, _, _, st = orc.grid_step(0.01, np.zeros(3), 0.0, R_REF, M_GRID, scen, -0.9,
                                             0.9, tlo, thi, j_star,
                                             workers=workers or orc.cpu_count())
        dt = time.perf_counter() - t0
        assert st["early_terms"] == 0 and feas and k == 1.0
        return dt

    def sequential(self, scen, n, j_star):
        """robust_rg_sequential (Alg. 2) on the same scenarios: one core, the reference's
        Python loop over scenarios (governor.py:496-504)."""
        if self.ref is not None:
            rf = self.ref
            cfg = rf.GovernorConfig(j_star=j_star, n_sim=n, n_kappa=8)
            box = rf.ConstraintSet(-0.9, 0.9, anchor=0.0)
            t0 = time.perf_counter()
            res = rf.robust_rg_sequential(rf.make_plant("surrogate-fc"), np.zeros(3),
                                          rf.GovernorState(0.0), R_REF, box, scen, cfg)
            dt = time.perf_counter() - t0
            assert res.kappa_opt == 1.0
            return dt
        import paper_2510_08288_b200 as rg
        orc = self.orc
        tlo, thi = orc.tighten(-0.9, 0.9, 0.0, 0.05)
        vlo, vhi = rg.admissible_setpoints(tlo, thi)
        t0 = time.perf_counter()
        kap = orc.bisect_all_c(0.01, np.zeros(3), 0.0, R_REF, -0.9, 0.9, vlo, vhi, scen,
                               j_star, 8)[0]
        dt = time.perf_counter() - t0
        assert np.all(kap == 1.0)
        return dt


def grid_sample_size(wl, spec, world):
    """Scenarios per reference step: the whole step for c2, a bounded sample of c4's
    2^20-scenario step (1/64 of it) so a step takes ~1 s on the host cores."""
    if wl == "c2":
        return spec["n_per_gpu"] * world
    return max(1, min(spec["n_total"], 16384))


def cpu_baseline(cpu: RefCPU, wl, spec, world, j_star, seconds):
    """Bounded CPU baseline on rank 0 (about `seconds` of timed work): the grid step on
    every core (best rep), one serial rep, and the sequential entry point."""
    if wl == "c1":
        return c1_cpu_baseline(cpu, j_star, seconds)
    if wl in ("c3", "c5"):
        return closed_loop_cpu_baseline(cpu, spec, j_star, seconds)
    n = grid_sample_size(wl, spec, world)
    cells = M_GRID * n * j_star
    pool = [cpu.scenarios(n, j_star, BASE_SEED + q) for q in range(4)]
    cpu.grid_step(pool[0], n, j_star)  # warm-up: JIT, thread pool, page faults
    times, t_end = [], time.perf_counter() + seconds
    while len(times) < 20 and (not times or time.perf_counter() < t_end):
        times.append(cpu.grid_step(pool[len(times) % 4], n, j_star))
    n_ser = min(n, 250)
    s_ser = cpu.scenarios(n_ser, j_star, BASE_SEED + 99)
    cpu.grid_step(s_ser, n_ser, j_star, workers=1)
    t_ser = cpu.grid_step(s_ser, n_ser, j_star, workers=1)
    n_seq = min(n, 1000)
    s_seq = pool[0] if n_seq == n else cpu.scenarios(n_seq, j_star, BASE_SEED + 98)
    cpu.sequential(s_seq, n_seq, j_star)
    t_seq = cpu.sequential(s_seq, n_seq, j_star)
    best = min(times)
    sample = (f"{len(times)} robust grid steps (M={M_GRID}, n_sim={n}, j*={j_star}, presampled "
              f"scenarios, the reference's kernel-only mode) on {cpu.cores()} threads, best rep")
    if wl == "c4":
        sample += f"; a {n}-scenario sample of the {spec['n_total']}-scenario step"
    return {
        "value": cells / best, "unit": UNIT, "cores": cpu.cores(), "kind": cpu.kind,
        "sample": sample, "ms_per_step": best * 1e3, "ms_per_step_mean": statistics.mean(times) * 1e3,
        "impl": cpu.info(),
        "serial_1core": {"value": M_GRID * n_ser * j_star / t_ser, "unit": UNIT,
                         "sample": f"1 step at n_sim={n_ser} (backend 'serial')"},
        "sequential_alg2_1core": {"ms_per_step": t_seq * 1e3, "n_sim": n_seq,
                                  "sample": "robust_rg_sequential on the step's scenarios, 1 core"},
    }


def c1_cpu_baseline(cpu: RefCPU, j_star, seconds):
    """C1 on the host: the reference's own functions in run_closed_loop's loop with
    bisection_rg at harness.py:200 (y_t, the governor step, plant.step + d_true from the
    reference's derive_seed(seed, "plant") stream), seed 2024, as many steps from t = 0 as
    fit in `seconds` (min 50), after 10 untimed steps (numba JIT)."""
    if cpu.ref is None:
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": "the C port has no closed-loop driver; c1 needs the reference"}
    rf = cpu.ref
    import refgov.disturbance as rdist
    setup = rf.load_config({})
    plant, cset, cfg = setup.plant, setup.cset, setup.governor
    lo = np.array([a for a, _ in setup.model.ranges])
    span = np.array([b - a for a, b in setup.model.ranges])

    def loop(steps):
        d_true = lo + span * rdist._uniform_grid(rdist.derive_seed(setup.seed, "plant"), 1, steps,
                                                 setup.model.state_dim)[0]
        r_sched = setup.profile.schedule(steps)
        x, state, cells = np.zeros(plant.state_dim), rf.GovernorState(v_prev=0.0), 0
        t0 = time.perf_counter()
        for t in range(steps):
            plant.output(x, state.v_prev)
            res = rf.bisection_rg(plant, x, state, float(r_sched[t]), cset, cfg)
            cells += int(res.diagnostics.get("sims_run", 0))
            x = plant.step(x, res.v_applied) + d_true[t]
        return time.perf_counter() - t0, cells

    loop(10)
    t_probe, _ = loop(50)
    steps = max(50, min(2000, int(seconds / max(t_probe / 50, 1e-6))))
    dt, cells = loop(steps)
    return {"value": cells * j_star / dt, "unit": UNIT, "cores": 1, "kind": cpu.kind,
            "steps": steps, "ms_per_closed_loop_step": dt * 1e3 / steps,
            "sample": f"1 episode (seed {setup.seed}) x {steps} closed-loop steps from t = 0: "
                      "refgov.bisection_rg + plant.step per step (the reference's Python loop, one "
                      "core)", "impl": cpu.info()}


def closed_loop_cpu_baseline(cpu: RefCPU, spec, j_star, seconds):
    """C3 / C5 on the host: the reference's run_closed_loop for one episode (seed 2024) at
    spec n_sim scenarios from t = 0, as many closed-loop steps as fit in `seconds` (min 2),
    after one untimed step (numba JIT, thread pool)."""
    n = spec["n_sim"]
    if cpu.ref is None:
        return {"value": None, "unit": UNIT, "cores": cpu.cores(), "kind": "port",
                "sample": "the C port has no closed-loop driver; c3 / c5 need the reference"}
    rf = cpu.ref
    setup = rf.load_config({"governor": {"n_sim": n, "backend": "multicore"}})
    t0 = time.perf_counter()
    rf.run_closed_loop(setup.plant, setup.cset, setup.model, setup.governor, setup.profile, 1,
                       setup.seed)
    t_one = time.perf_counter() - t0
    steps = max(2, int(seconds / max(t_one, 1e-3)))
    t0 = time.perf_counter()
    rec = rf.run_closed_loop(setup.plant, setup.cset, setup.model, setup.governor,
                             setup.profile, steps, setup.seed)
    dt = time.perf_counter() - t0
    sims = sum(int(d.split(",")[4]) for d in getattr(rec, "diag_rows", [])) if \
        getattr(rec, "diag_rows", None) else None
    cells = (sims * j_star) if sims else None
    return {"value": (cells / dt) if cells else None, "unit": UNIT, "cores": cpu.cores(),
            "kind": cpu.kind, "steps": steps, "ms_per_closed_loop_step": dt * 1e3 / steps,
            "episode_steps_per_s": steps / dt,
            "sample": f"1 episode (seed {setup.seed}) x {steps} closed-loop steps at n_sim={n} "
                      "through refgov.run_closed_loop (host sampling included, as the reference "
                      "runs it)", "impl": cpu.info()}


REF_BUDGET_S = 150.0  # the reference arm stops timing after this many seconds of steps


def run_reference(args, rank, world, wl, spec):
    """The reference's CPU path on the host cores, rank 0 only: W untimed steps, then up
    to K timed steps (each a bounded sample of the workload), stopping early once
    REF_BUDGET_S seconds are spent so the arm ends within a few minutes."""
    if rank != 0:
        return
    cpu = RefCPU()
    j_star = args.j_star
    config = config_of(wl, spec, world, j_star)
    if wl in ("c1", "c3", "c5"):
        cb = c1_cpu_baseline(cpu, j_star, min(REF_BUDGET_S, 20.0)) if wl == "c1" else \
            closed_loop_cpu_baseline(cpu, spec, j_star, min(REF_BUDGET_S, 40.0))
        value = cb["value"]
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
                "n_gpus": world, "steps": cb.get("steps"), "warmup": 1, "higher_is_better": True,
                "scaling": spec["scaling"], "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config, "cpu_baseline": cb,
                "ms_per_step": cb.get("ms_per_closed_loop_step"),
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    n = grid_sample_size(wl, spec, world)
    cells = M_GRID * n * j_star
    pool = [cpu.scenarios(n, j_star, BASE_SEED + q) for q in range(8)]  # outside the clock
    for s in range(max(args.warmup, 1)):
        cpu.grid_step(pool[s % 8], n, j_star)
    times, t_end = [], time.perf_counter() + REF_BUDGET_S
    for s in range(args.steps):
        times.append(cpu.grid_step(pool[s % 8], n, j_star))
        if time.perf_counter() > t_end:
            break
    total = float(sum(times))
    value = cells * len(times) / total
    sample = (f"{len(times)} timed robust grid steps (M={M_GRID}, n_sim={n}, j*={j_star}; "
              f"scenarios presampled outside the clock, the reference's kernel-only mode) on "
              f"{cpu.cores()} threads after {max(args.warmup, 1)} warm-up steps")
    if wl == "c4":
        sample += f"; each a {n}-scenario sample of the {spec['n_total']}-scenario step"
    cb = {"value": value, "unit": UNIT, "cores": cpu.cores(), "kind": cpu.kind,
          "sample": sample, "impl": cpu.info()}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": len(times), "steps_requested": args.steps,
        "warmup": args.warmup, "ms_per_step": total * 1e3 / len(times),
        "ms_per_step_full_workload": total * 1e3 / len(times) * (
            spec["n_total"] / n if wl == "c4" else 1.0),
        "higher_is_better": True, "scaling": spec["scaling"],
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ms_per_step_min": min(times) * 1e3,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- own arm: grid steps

def _vp():
    import ctypes
    return ctypes.c_void_p


def init_dist(world, local_rank):
    """torch.distributed for N>1 (NCCL, or gloo for the one-GPU smoke of the N>1 path),
    plus a gloo group whose barriers block in the kernel instead of spinning (used while
    rank 0 times the CPU baseline)."""
    import torch
    import torch.distributed as dist

    backend = os.environ.get("RG_BENCH_DIST_BACKEND", "nccl")
    if "WORLD_SIZE" not in os.environ:  # RG_BENCH_FORCE_DIST at world size 1, no torchrun
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0",
                          WORLD_SIZE="1", LOCAL_RANK="0")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        dist.init_process_group(backend)
    cpu_group = dist.new_group(backend="gloo") if backend == "nccl" else None
    return backend, cpu_group


def run_own(args, rank, world, local_rank, wl, spec):
    import torch

    if "RG_BENCH_DEVICE" in os.environ:
        local_rank = int(os.environ["RG_BENCH_DEVICE"])
    torch.cuda.set_device(local_rank)
    backend, cpu_group = (None, None)
    if MULTI:
        backend, cpu_group = init_dist(world, local_rank)
    if wl == "c5":
        line = run_c5(args, rank, world, local_rank, spec, backend, cpu_group)
    elif wl == "c3":
        line = run_c3(args, rank, world, local_rank, spec, backend, cpu_group)
    elif wl == "c1":
        line = run_c1(args, rank, world, local_rank, spec, backend, cpu_group)
    else:
        line = run_grid(args, rank, world, local_rank, wl, spec, backend, cpu_group)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if MULTI:
        torch.distributed.destroy_process_group()


def _max_over_ranks(x: float, world, device) -> float:
    if not MULTI:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def run_grid(args, rank, world, local_rank, wl, spec, backend, cpu_group):
    import torch

    import paper_2510_08288_b200 as rg
    from paper_2510_08288_b200 import _capi

    dev = f"cuda:{local_rank}"
    ctx = _capi.context(local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda", local_rank))
    j_star = args.j_star
    if wl == "c2":
        n_total = spec["n_per_gpu"] * world
        k0, n_rank = rank * spec["n_per_gpu"], spec["n_per_gpu"]
    else:
        n_total = spec["n_total"]
        k0 = rank * n_total // world
        n_rank = (rank + 1) * n_total // world - k0
    cells_rank = M_GRID * n_rank * j_star
    cells_step = M_GRID * n_total * j_star
    plant = rg.make_plant("surrogate-fc")
    box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
    tight = rg.tighten(box, 0.05)
    v_lo, v_hi = rg.admissible_setpoints(tight.lower, tight.upper)
    prob = _capi.Problem(0.01, -0.9, 0.9, v_lo, v_hi, j_star, 0)
    model = rg.DisturbanceModel.scaled(0.001, 3)
    x0 = np.zeros(3)
    lib = ctx.lib
    res = _capi.GridResult()
    viol = torch.zeros(M_GRID, dtype=torch.int32, device=dev)
    flags = _capi.RG_ASYNC | _capi.RG_NO_TIMING
    if MULTI:
        flags |= _capi.RG_DEVICE_PTRS
    x0_ptr = x0.ctypes.data_as(_vp())  # kernel parameter: host memory
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    row_idx = torch.arange(M_GRID, dtype=torch.int32, device=dev)
    minus1 = torch.full_like(row_idx, -1)
    dist = torch.distributed if MULTI else None

    p2p = MULTI and args.xchg == "p2p"
    if p2p:  # the exchange fused into the step kernel: no collective call per step
        from paper_2510_08288_b200.sharded import _p2p_ready
        _p2p_ready(ctx, dist, None)
        flags |= _capi.RG_XCHG

    def launch(s):
        scen = _capi.make_scenarios(BASE_SEED + s, k0, n_rank, model.lo, model.span)
        _capi.check(lib.rg_grid_step(ctx.handle, prob, x0_ptr, 0.0, R_REF, M_GRID, 0, None,
                                     n_rank, 0, scen,
                                     _vp()(viol.data_ptr()) if MULTI and not p2p else None,
                                     None, res, flags))

    def exchange():
        if p2p:  # done inside the kernel; the global row is in the step's result block
            return None
        # per-row violating-scenario counts, int32 (a gated-out row is -1 on every rank):
        # the global MAX is 0 exactly for the rows feasible on every shard
        dist.all_reduce(viol, op=dist.ReduceOp.MAX)
        return torch.where(viol == 0, row_idx, minus1).max()  # literal Eq. 4

    with torch.cuda.stream(stream):
        for s in range(args.warmup):
            launch(s)
            if MULTI:
                exchange()
        torch.cuda.synchronize()
        if MULTI:
            dist.barrier()
        sampler = ClockSampler(local_rank)
        sampler.start()
        time.sleep(0.2)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)]
              for _ in range(args.steps)]
        best_rows = []
        torch.cuda.synchronize()
        if MULTI:
            dist.barrier()
        # The timed steps are enqueued in chunks behind a device-side sleep, so the device
        # never idles waiting for the host to submit the next step inside an event pair.
        wall = 0.0
        for c0 in range(0, args.steps, CHUNK):
            c1 = min(args.steps, c0 + CHUNK)
            if not MULTI:
                torch.cuda._sleep(int(SLEEP_CYCLES_PER_STEP * (c1 - c0)))
            w0 = time.perf_counter()
            for s in range(c0, c1):
                flush.zero_()  # L2 flush between timed steps, outside the events
                ev[s][0].record(stream)
                launch(args.warmup + s)
                ev[s][1].record(stream)
                if MULTI:
                    best_rows.append(exchange())
                ev[s][2].record(stream)
            torch.cuda.synchronize()
            wall += time.perf_counter() - w0
        if MULTI:
            dist.barrier()
        clocks = sampler.stop()
    per = np.array([a.elapsed_time(c) for a, _, c in ev])  # ms, whole step
    kern = np.array([a.elapsed_time(b) for a, b, _ in ev])  # ms, generator + grid kernels
    xch = per - kern
    total_ms = _max_over_ranks(float(per.sum()), world, dev)
    kernel_ms = _max_over_ranks(float(kern.mean()), world, dev)
    # the step's decision must be the reference's: all 32 rows feasible -> kappa = 1
    if not MULTI or p2p:
        out = _capi.GridResult()
        _capi.check(lib.rg_grid_fetch(ctx.handle, None, M_GRID, out))
        assert out.row == M_GRID - 1, out.row
        assert p2p or out.early_terms == 0, out.early_terms
    else:
        assert all(int(b.item()) == M_GRID - 1 for b in best_rows[-3:])

    # k_gen_soa + k_grid when the scenario block is staged, k_grid alone when fused
    launches_per_step = 2 if n_rank * j_star * 24 <= (16 << 30) else 1
    value = cells_step * args.steps / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps

    # dominant kernel: k_grid.  The events bracket k_gen_soa + k_grid; the ncu launch list
    # (profiles/) gives k_grid's share.
    peak = ctx.fp64_peak()
    achieved = FLOPS_PER_CELL_STEP * cells_rank / (kernel_ms * 1e-3)
    fp64_per_cell = _ncu_summary().get("fp64_instr_per_cell_step", FP64_INSTR_PER_CELL_STEP)
    fp64_instr_rate = cells_rank / (kernel_ms * 1e-3) * fp64_per_cell
    roof = {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12,
            "unit": "TFLOP/s", "frac": achieved / peak, "traffic": _ncu_traffic(n_rank),
            "fp64_pipe_frac": fp64_instr_rate / (peak / 2.0),
            "issue_model": issue_model(n_rank, j_star, kernel_ms, clocks),
            "fp64_instr_per_cell_step": fp64_per_cell,
            "peak_source": "measured in this run: rg_fp64_peak (independent DFMA chains, "
                           "2 flop per DFMA); MEASURED_PEAKS.json has no FP64 figure",
            "flops_per_cell_step": FLOPS_PER_CELL_STEP, "cell_steps_per_launch": cells_rank,
            "kernel_ms": kernel_ms,
            "kernel_timing": "CUDA events around k_gen_soa + k_grid on the library's stream "
                             "(per rank; the max over ranks)"}

    e2e = None
    if args.e2e_steps > 0:
        e2e = e2e_grid(args, rank, world, local_rank, rg, plant, box, model, n_total, n_rank,
                       j_star, dev)

    latency = None
    if not MULTI:
        latency = latency_split(ctx, lib, prob, x0_ptr, model, k0, n_rank)
    else:
        latency = {"allreduce_us_p50": float(np.median(xch) * 1e3),
                   "allreduce_us_p90": float(np.percentile(xch, 90) * 1e3),
                   "kernel_us_p50": float(np.median(kern) * 1e3),
                   "note": "per step on rank 0: kernel = k_gen_soa + k_grid (events), "
                           f"allreduce = the {backend} all-reduce (MAX) of the int32[32] row "
                           "counts plus the on-device row extraction, including any wait for "
                           "the slowest rank"}

    sweep = []
    if not MULTI and not args.no_sweep:
        sweep = run_sweep(args, ctx, lib, stream, flush, prob, x0, x0_ptr, model, plant, box,
                          rg, _capi, res, flags, j_star, n_rank, peak, clocks, torch)
    one_gpu = None
    if MULTI and wl == "c4" and rank == 0:
        # the whole c4 step on rank 0's GPU alone (no shard, no exchange), same run: the
        # one-GPU point of this workload, beside the N-GPU value
        ts = []
        with torch.cuda.stream(stream):
            for s_i in range(4):
                flush.zero_()
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                sc = _capi.make_scenarios(BASE_SEED + 77 + s_i, 0, n_total, model.lo, model.span)
                _capi.check(lib.rg_grid_step(ctx.handle, prob, x0_ptr, 0.0, R_REF, M_GRID, 0, None,
                                             n_total, 0, sc, None, None, res,
                                             _capi.RG_ASYNC | _capi.RG_NO_TIMING))
                b_.record(stream)
                torch.cuda.synchronize()
                if s_i:
                    ts.append(a_.elapsed_time(b_))
        one_gpu = {"n_sim": n_total, "ms_per_step": float(np.mean(ts)),
                   "value": cells_step / (float(np.mean(ts)) * 1e-3), "unit": UNIT,
                   "note": "the same c4 step, all 2^20 scenarios on rank 0's GPU alone, measured "
                           "in this run after the timed region (3 steps after 1 warm-up)"}

    cb = None
    if MULTI:
        torch.distributed.barrier()
    if rank == 0 and not args.no_cpu_baseline:
        cb = cpu_baseline(RefCPU(), wl, spec, world, j_star, args.cpu_seconds)
    if MULTI:
        torch.distributed.barrier(group=cpu_group)  # gloo: the other ranks block, not spin

    par = f"scenario shards x{world}" + (
        f", {backend} all-reduce (MAX) of the int32[{M_GRID}] row counts per step, row "
        "extracted on every device" if MULTI and not p2p else "") + (
        ", the row counts exchanged inside the step kernel over NVLink (RG_XCHG), row "
        "extracted on every device" if p2p else "")
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": spec["scaling"], "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config_of(wl, spec, world, j_star),
        "parallelism": par,
        "run": {"rng": ("staged (k_gen_soa + k_grid)" if launches_per_step == 2
                        else "fused (k_grid)"),
                "n_sim_per_gpu": n_rank, "cell_steps_per_step": cells_step,
                "dist_backend": backend},
        "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "latency": latency,
        "sweep": sweep, "c4_one_gpu_same_run": one_gpu,
        "gpu_launches": args.steps * launches_per_step, "clocks": clocks,
        "host_enqueue_ms_per_step": wall * 1e3 / args.steps,
        "kernel_ms_p50": float(np.median(kern)), "step_ms_p50": float(np.median(per)),
        "step_ms_min": float(per.min()),
    }


def e2e_grid(args, rank, world, local_rank, rg, plant, box, model, n_total, n_rank, j_star,
             dev):
    """The same step through the public API with host inputs, the result on the host."""
    import torch

    if not MULTI:
        cfg = rg.GovernorConfig(j_star=j_star, m_grid=M_GRID, n_sim=n_rank, device=local_rank)
        for s in range(5):
            rg.robust_rg_parallel(plant, np.zeros(3), rg.GovernorState(0.0), R_REF, box,
                                  rg.sample_scenarios(model, n_rank, j_star + 1, seed=s,
                                                      device=local_rank), cfg)
        t0 = time.perf_counter()
        for s in range(args.e2e_steps):
            scen = rg.sample_scenarios(model, n_rank, j_star + 1, seed=BASE_SEED + s,
                                       device=local_rank)
            r = rg.robust_rg_parallel(plant, np.zeros(3), rg.GovernorState(0.0), R_REF, box,
                                      scen, cfg)
        t_e2e = (time.perf_counter() - t0) / args.e2e_steps
        assert r.kappa_opt == 1.0 and r.matrix.all()
        h2d = 3 * 8 + 2 * 8 + 9 * 8   # x0, v_prev/r, scenario stream descriptor (kernel params)
        d2h = (M_GRID * ((n_rank + 31) // 32) * 4) + M_GRID * 4 + 64  # P bits, counts, result
        return {"value": M_GRID * n_rank * j_star / t_e2e, "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e * 1e3,
                "api": "paper_2510_08288_b200.robust_rg_parallel (keep_matrix=True: P returned)"}
    from paper_2510_08288_b200.sharded import robust_rg_parallel_sharded
    cfg = rg.GovernorConfig(j_star=j_star, m_grid=M_GRID, n_sim=n_total, device=local_rank)
    for s in range(2):
        robust_rg_parallel_sharded(plant, np.zeros(3), rg.GovernorState(0.0), R_REF, box,
                                   rg.sample_scenarios(model, n_total, j_star + 1, seed=s,
                                                       device=local_rank), cfg,
                                   exchange=args.xchg)
    torch.distributed.barrier()
    t0 = time.perf_counter()
    for s in range(args.e2e_steps):
        scen = rg.sample_scenarios(model, n_total, j_star + 1, seed=BASE_SEED + s,
                                   device=local_rank)
        r = robust_rg_parallel_sharded(plant, np.zeros(3), rg.GovernorState(0.0), R_REF, box,
                                       scen, cfg, exchange=args.xchg)
    t_e2e = _max_over_ranks((time.perf_counter() - t0) / args.e2e_steps, world, dev)
    assert r.kappa_opt == 1.0
    return {"value": M_GRID * n_total * j_star / t_e2e, "unit": UNIT,
            "h2d_bytes_per_step": 112, "d2h_bytes_per_step": M_GRID * 4,
            "ms_per_step": t_e2e * 1e3,
            "api": f"paper_2510_08288_b200.sharded.robust_rg_parallel_sharded(exchange="
                   f"{args.xchg!r}) (every rank returns the KappaResult; wall clock, max over "
                   "ranks)"}


def latency_split(ctx, lib, prob, x0_ptr, model, k0, n_sim):
    """One synchronous step through the C ABI (no P): host call -> result in host memory,
    the device span of k_grid (first block start to publication, globaltimer) and the
    final reduction inside it."""
    from paper_2510_08288_b200 import _capi

    sync_res = _capi.GridResult()
    walls, spans, reds = [], [], []
    for s in range(220):
        scen = _capi.make_scenarios(BASE_SEED + 20000 + s, k0, n_sim, model.lo, model.span)
        t0 = time.perf_counter()
        _capi.check(lib.rg_grid_step(ctx.handle, prob, x0_ptr, 0.0, R_REF, M_GRID, 0, None,
                                     n_sim, 0, scen, None, None, sync_res, _capi.RG_NO_TIMING))
        dt = time.perf_counter() - t0
        if s >= 20:
            walls.append(dt * 1e6)
            spans.append(sync_res.kernel_ms * 1e3)
            reds.append(sync_res.reduce_us)
    return {"api_call_us": float(np.median(walls)),
            "k_grid_span_us": float(np.median(spans)),
            "launch_overhead_us": float(np.median(walls) - np.median(spans)),
            "reduction_us": float(np.median(reds)),
            "note": "median of 200 synchronous rg_grid_step calls at the workload (no P): "
                    "api_call = host wall time of the call; k_grid_span = first block start "
                    "to result publication (device globaltimer); launch_overhead = the "
                    "difference (host enqueue, launch latency, k_gen_soa, result visibility); "
                    "reduction = the last block's row extraction and publication inside the span"}


def run_sweep(args, ctx, lib, stream, flush, prob, x0, x0_ptr, model, plant, box, rg, _capi,
              res, flags, j_star, n_sim, peak, clocks, torch):
    """Other sizes and entry points at N=1 (reported beside the headline, not in it)."""
    sweep = []
    for n_big, reps in ((10_000, 20), (1 << 20, 3)):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(reps + 1)]
        with torch.cuda.stream(stream):
            for s_i, (a, b) in enumerate(evs):
                flush.zero_()
                a.record(stream)
                sc = _capi.make_scenarios(BASE_SEED + 1000 + s_i, 0, n_big, model.lo, model.span)
                _capi.check(lib.rg_grid_step(ctx.handle, prob, x0_ptr, 0.0, R_REF, M_GRID, 0,
                                             None, n_big, 0, sc, None, None, res, flags))
                b.record(stream)
            torch.cuda.synchronize()
        t = np.array([a.elapsed_time(b) for a, b in evs[1:]])
        cells = M_GRID * n_big * j_star
        rate = cells / (t.mean() * 1e-3)
        sweep.append({"n_sim": n_big, "ms_per_step": float(t.mean()), "value": rate,
                      "unit": UNIT, "roofline_frac": FLOPS_PER_CELL_STEP * rate / peak,
                      "issue_frac": issue_model(n_big, j_star, float(t.mean()), clocks)["frac"],
                      "rng": "staged" if n_big * j_star * 24 <= (16 << 30) else "fused"})

    # dense host scenario tensor (the reference API's normal input, ScenarioSet(data)):
    # 24.7 bytes per scenario-step copied host -> device inside every call
    cfg = rg.GovernorConfig(j_star=j_star, m_grid=M_GRID, n_sim=n_sim)
    dense = [rg.ScenarioSet(rg.sample_scenarios(model, n_sim, j_star + 1, seed=40 + q).data,
                            seed=40 + q, model=model) for q in range(4)]
    for q in range(4):
        rg.robust_rg_parallel(plant, x0, rg.GovernorState(0.0), R_REF, box, dense[q], cfg)
    t0 = time.perf_counter()
    for q in range(40):
        r = rg.robust_rg_parallel(plant, x0, rg.GovernorState(0.0), R_REF, box, dense[q % 4], cfg)
    t_d = (time.perf_counter() - t0) / 40
    assert r.kappa_opt == 1.0
    sweep.append({"workload": f"e2e with a dense host ScenarioSet (n_sim={n_sim}, "
                              f"{dense[0].data.nbytes} B host->device per call)",
                  "ms_per_step": t_d * 1e3, "value": M_GRID * n_sim * j_star / t_d, "unit": UNIT,
                  "timing": "wall clock around robust_rg_parallel (P returned)"})

    # C5 shape: a batch of independent episodes in one launch (64 x 10k scenarios, bench
    # snapshot so every row runs the full horizon), and C3: the desk-scale closed loop at
    # 10k scenarios (the whole 2000-step trace)
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
    # the bisection searches: Alg. 2 on the C2 step itself (r = 0.5: one feasible rollout
    # per scenario), then a transient step (r = 2.5 from rest, kappa* = 0.5078): exact Alg. 2
    # (per-scenario bisections, min) and the joint search (one kappa for all scenarios per
    # iteration, OR-reduced flag); both land on the same kappa
    sc = _capi.make_scenarios(BASE_SEED, 0, n_sim, model.lo, model.span)
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
                ("joint", lambda: ctx.bisect_joint(prob, x0, 0.0, 2.5, 8, None, n_b, sc)),
                ("joint, one launch per iteration",
                 lambda: ctx.bisect_joint(prob, x0, 0.0, 2.5, 8, None, n_b, sc,
                                          per_iteration=True))):
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
    return sweep


# ---------------------------------------------------------------- own arm: C5 episodes

def active_cells(V_prev, R, m_grid, interval):
    """Per episode, the reference's sims_run / n_sim for one grid step (governor.py:302-317,
    341): candidate rows that pass the steady-state gate, duplicates counted once.
    Vectorised restatement of _host_rows over episodes (same three roundings)."""
    kap = np.arange(m_grid, dtype=np.float64) / (m_grid - 1)
    V = V_prev[:, None] + kap[None, :] * (R - V_prev)[:, None]
    V[:, 0] = V_prev
    V[:, -1] = R
    lo, hi = interval
    ok = (V >= lo) & (V <= hi)
    Vs = np.where(ok, V, np.nan)
    Vs.sort(axis=1)
    distinct = np.isfinite(Vs) & np.concatenate(
        [np.ones((Vs.shape[0], 1), bool), Vs[:, 1:] != Vs[:, :-1]], axis=1)
    return distinct.sum(axis=1)


def run_c1(args, rank, world, local_rank, spec, backend, cpu_group):
    """C1 (configs[0]): the desk-scale closed loop with the nominal bisection governor through
    the public API (run_closed_loop_bisection -> rg_closed_loop_bisection: the whole trace as
    one device kernel, k_loop_bisect).  W untimed steps of another episode, then the timed
    episode from t = 0 for K steps; host wall clock of the whole loop, the max over ranks.
    Cell-steps = the rollouts (sims_run) x j* summed over the timed steps."""
    import torch

    import paper_2510_08288_b200 as rg
    from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop_bisection

    dev = f"cuda:{local_rank}"
    j_star = args.j_star
    plant = rg.make_plant("surrogate-fc")
    box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
    model = rg.DisturbanceModel.scaled(0.001, 3)
    cfg = rg.GovernorConfig(j_star=j_star, n_kappa=8, device=local_rank)
    prof = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
    seed = 2024 + rank
    if args.warmup > 0:
        run_closed_loop_bisection(plant, box, model, cfg, prof, args.warmup, seed + 1000)
    torch.cuda.synchronize()
    if MULTI:
        torch.distributed.barrier()
    from paper_2510_08288_b200 import _capi

    ctx = _capi.context(local_rank)
    sampler = ClockSampler(local_rank)
    sampler.start()
    t0 = time.perf_counter()
    out = run_closed_loop_bisection(plant, box, model, cfg, prof, args.steps, seed)
    wall = time.perf_counter() - t0
    clocks = sampler.stop()
    cells = sum(int(r.diagnostics["sims_run"]) for r, _ in out)
    total = _max_over_ranks(wall, world, dev)
    if MULTI:
        t = torch.tensor([cells], dtype=torch.int64, device=dev)
        torch.distributed.all_reduce(t)
        cells = int(t.item())
    value = cells * j_star / total
    roof = wall_roofline(value / world, local_rank,
                         "host wall clock of the closed loop per GPU (one device kernel for the "
                         "trace): a lower bound on the kernel's rate")
    cb = None
    if MULTI:
        torch.distributed.barrier()
    if rank == 0 and not args.no_cpu_baseline:
        cb = c1_cpu_baseline(RefCPU(), j_star, min(args.cpu_seconds, 20.0))
    if MULTI:
        torch.distributed.barrier(group=cpu_group)
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total * 1e3 / args.steps,
        "higher_is_better": True, "scaling": spec["scaling"], "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": config_of("c1", spec, world, j_star),
        "parallelism": f"one closed-loop episode per GPU x{world} (replicas)",
        "run": {"found_steps": sum(1 for r, _ in out if r.feasible),
                "rollouts_total": cells,
                "timing": "host wall clock of the whole timed closed loop, max over ranks"},
        # per step r_t and d_true[t] in (32 B); kappa, v, y, cells, early, device ns and the
        # found flag out (49 B), copied once around the one launch
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 32, "d2h_bytes_per_step": 49,
                "note": "the timed loop is the public API end to end: run_closed_loop_bisection "
                        "-> rg_closed_loop_bisection (one device kernel for the whole trace)"},
        "roofline": roof, "cpu_baseline": cb, "clocks": clocks, "gpu_launches": 1,
    }


def run_c3(args, rank, world, local_rank, spec, backend, cpu_group):
    """C3: the reference's desk-scale closed loop (harness.py:138-224) at n_sim scenarios per
    step through the public API (run_closed_loop: rg_closed_loop, which runs the whole trace
    as one cooperative kernel, k_loop_ts -- every governor step on the time-split form, the
    row, kappa, v_t and the true plant with numpy's tanh restated on the device between grid
    barriers; with RG_NO_DEVICE_LOOP=1 one grid-step launch per closed-loop step and the
    plant on the host).  W untimed closed-loop steps of another episode (seed + 1000), then
    the timed episode from t = 0 for K steps; host wall clock of the whole loop (it is the
    latency a controller sees: sampling descriptor, device step, result, plant update), the
    max over ranks.  Cell-steps = the reference's sims_run x j* summed over the timed steps."""
    import torch

    import paper_2510_08288_b200 as rg
    from paper_2510_08288_b200.harness import ReferenceProfile, run_closed_loop

    dev = f"cuda:{local_rank}"
    n, j_star = spec["n_sim"], args.j_star
    plant = rg.make_plant("surrogate-fc")
    box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
    model = rg.DisturbanceModel.scaled(0.001, 3)
    cfg = rg.GovernorConfig(j_star=j_star, m_grid=M_GRID, n_sim=n, device=local_rank)
    prof = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
    seed = 2024 + rank
    if args.warmup > 0:
        run_closed_loop(plant, box, model, cfg, prof, args.warmup, seed + 1000)
    torch.cuda.synchronize()
    if MULTI:
        torch.distributed.barrier()
    from paper_2510_08288_b200 import _capi

    ctx = _capi.context(local_rank)
    launches0 = ctx.get_option("grid_step_kernels")
    sampler = ClockSampler(local_rank)
    sampler.start()
    t0 = time.perf_counter()
    rec = run_closed_loop(plant, box, model, cfg, prof, args.steps, seed)
    wall = time.perf_counter() - t0
    clocks = sampler.stop()
    # counted by the library: the step kernel per step (the time-split step generates its
    # own scenarios), plus the generator where a step staged its block
    launches = ctx.get_option("grid_step_kernels") - launches0
    device_loop = bool(ctx.get_option("last_loop_device"))
    assert not rec.aborted
    sims = sum(int(d.split(",")[4]) for d in rec.diag_rows)
    total = _max_over_ranks(wall, world, dev)
    if MULTI:
        t = torch.tensor([sims], dtype=torch.int64, device=dev)
        torch.distributed.all_reduce(t)
        sims = int(t.item())
    value = sims * j_star / total
    roof = wall_roofline(value / world, local_rank,
                         "host wall clock of the closed loop per GPU (device step, result "
                         "readback, host true-plant step): a lower bound on the kernels' rate")
    cb = None
    if MULTI:
        torch.distributed.barrier()
    if rank == 0 and not args.no_cpu_baseline:
        cb = closed_loop_cpu_baseline(RefCPU(), spec, j_star, args.cpu_seconds)
    if MULTI:
        torch.distributed.barrier(group=cpu_group)
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total * 1e3 / args.steps,
        "higher_is_better": True, "scaling": spec["scaling"], "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": config_of("c3", spec, world, j_star),
        "parallelism": f"one closed-loop episode per GPU x{world} (replicas)",
        "run": {"violations": rec.violations(box), "sims_run_total": sims,
                "active_rows_mean": sims / (n * args.steps * world),
                "timing": "host wall clock of the whole timed closed loop (device governor step, "
                          "host true-plant step, result readback), max over ranks"},
        # device loop: per step r_t and d_true[t] in (32 B) and v, kappa, y, sims, early,
        # device ns and the feasible flag out (49 B), copied once around the one launch.
        # Per-step loop: the state, v_prev and r travel as kernel parameters (5 doubles)
        # beside the RNG descriptor and the host row plan (112 B); the result block (128 B
        # header + M row words) is written by the kernel into pinned host memory.  The loop
        # never reads P, so run_closed_loop asks for none (the reference's diagnostics stay).
        "e2e": {"value": value, "unit": UNIT,
                "h2d_bytes_per_step": 32 if device_loop else 5 * 8 + 112,
                "d2h_bytes_per_step": 49 if device_loop else 128 + 4 * M_GRID,
                "note": "the timed loop is the public API end to end: run_closed_loop -> "
                        "rg_closed_loop, " + (
                            "the whole trace as one cooperative kernel (k_loop_ts: grid step, "
                            "row, kappa, v_t and the true plant with numpy's tanh restated, on "
                            "the device)" if device_loop else
                            "one grid step launch per closed-loop step, then kappa, v_t and "
                            "the true plant on the host")},
        "device_loop": device_loop,
        "roofline": roof, "cpu_baseline": cb, "clocks": clocks, "gpu_launches": launches,
    }


def run_c5(args, rank, world, local_rank, spec, backend, cpu_group):
    """C5: the desk-scale closed loop for E episodes (seeds 2024 + e) at n_sim scenarios,
    episodes split over the ranks (replicas, no collective on the data path).  W closed-loop
    steps untimed, then K timed steps (each: one batched governor launch per rank + the
    vectorised true-plant step on the host), max over ranks."""
    import torch

    import paper_2510_08288_b200 as rg
    from paper_2510_08288_b200.harness import ReferenceProfile, _rk4_batch
    from paper_2510_08288_b200.disturbance import derive_seed

    dev = f"cuda:{local_rank}"
    E_total, n, j_star = spec["episodes"], spec["n_sim"], args.j_star
    e0, e1 = rank * E_total // world, (rank + 1) * E_total // world
    seeds = np.arange(2024 + e0, 2024 + e1)
    E = seeds.size
    plant = rg.make_plant("surrogate-fc")
    box = rg.ConstraintSet(-0.9, 0.9, anchor=0.0)
    model = rg.DisturbanceModel.scaled(0.001, 3)
    cfg = rg.GovernorConfig(j_star=j_star, m_grid=M_GRID, n_sim=n, device=local_rank)
    prof = ReferenceProfile(((0, 0.4), (400, 2.5), (1000, -2.5), (1600, 0.2)))
    T = args.warmup + args.steps
    R = np.tile(prof.schedule(T), (E, 1))
    scen_seeds = [derive_seed(int(s), "scenarios") for s in seeds]
    # the true-plant disturbance stream of every episode (harness.py:172-174)
    D = np.stack([rg.sample_scenarios(model, 1, T, derive_seed(int(s), "plant"),
                                      device=local_rank).data[0] for s in seeds])
    tight = rg.tighten(box, 0.05)
    interval = rg.admissible_setpoints(tight.lower, tight.upper)
    X = np.zeros((E, 3))
    Vp = np.zeros(E)

    def step(t):
        kap, v, feas, _ = rg.robust_rg_parallel_batch(
            plant, X, Vp, R[:, t], box, model, n, [s + t for s in scen_seeds], cfg)
        act = active_cells(Vp, R[:, t], M_GRID, interval)
        Xn = _rk4_batch(plant.step_size, X, v) + D[:, t]
        return v, Xn, act

    for t in range(args.warmup):
        v, X, _ = step(t)
        Vp = v
    torch.cuda.synchronize()
    if MULTI:
        torch.distributed.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    times, acts = [], 0
    for t in range(args.warmup, T):
        t0 = time.perf_counter()
        v, X, act = step(t)
        times.append(time.perf_counter() - t0)
        Vp = v
        acts += int(act.sum())
    clocks = sampler.stop()
    total = _max_over_ranks(sum(times), world, dev)
    acts_all = acts
    if MULTI:
        t = torch.tensor([acts], dtype=torch.int64, device=dev)
        torch.distributed.all_reduce(t)
        acts_all = int(t.item())
    cells = acts_all * n * j_star  # the reference's sims_run x j* over all episodes and steps
    value = cells / total
    ms = total * 1e3 / args.steps
    roof = wall_roofline(value / world, local_rank,
                         "host wall clock per GPU of the batched governor call (host compaction, "
                         "copies, k_grid_pairs) plus the host true-plant step",
                         _ncu_summary("r02_k_grid_pairs_512_ncu.json"))
    cb = None
    if MULTI:
        torch.distributed.barrier()
    if rank == 0 and not args.no_cpu_baseline:
        cb = closed_loop_cpu_baseline(RefCPU(), spec, j_star, args.cpu_seconds)
    if MULTI:
        torch.distributed.barrier(group=cpu_group)
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": spec["scaling"], "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": config_of("c5", spec, world, j_star),
        "parallelism": f"episode replicas: {E_total // world}-{-(-E_total // world)} episodes "
                       f"per GPU x{world}, no collective on the data path",
        "run": {"episodes_per_gpu": E, "closed_loop_steps_timed": args.steps,
                "first_timed_t": args.warmup, "active_rows_mean": acts_all / (E_total * args.steps),
                "cell_steps_counted": "active rows (gate + dedup, the reference's sims_run / "
                                      "n_sim) x n_sim x j* per episode-step"},
        "episode_steps_per_s": E_total * args.steps / total,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": E_total * 6 * 8,
                "d2h_bytes_per_step": E_total * 28,
                "note": "the timed loop already runs through the public API "
                        "(robust_rg_parallel_batch) with host inputs and host results"},
        "roofline": roof, "cpu_baseline": cb, "clocks": clocks,
        "gpu_launches": args.steps,
    }


# ---------------------------------------------------------------- ncu summaries

def wall_roofline(rate_per_gpu, device, timing, ncu=None):
    """The FP64 roofline fraction of a wall-clock rate (closed loops: the host is in the loop)."""
    from paper_2510_08288_b200 import _capi

    peak = _capi.context(device).fp64_peak()
    achieved = FLOPS_PER_CELL_STEP * rate_per_gpu
    out = {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
           "frac": achieved / peak, "traffic": (ncu or {}).get("dram_bytes_per_launch"),
           "flops_per_cell_step": FLOPS_PER_CELL_STEP, "timing": timing,
           "peak_source": "measured in this run: rg_fp64_peak (independent DFMA chains)"}
    if ncu:
        out["ncu"] = {k: ncu.get(k) for k in ("workload", "fp64_instr_per_cell_step",
                                               "instr_per_cell_step", "fp64_pipe_pct_of_peak")}
    return out


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


def _ncu_traffic(n_sim=1000):
    """dram bytes per k_grid launch from the committed ncu --set full summary of the
    nearest size (C2 or 10k)."""
    return (_ncu_summary() if n_sim <= 1000 else
            _ncu_summary("k_grid_ncu_10k.json")).get("dram_bytes_per_launch")


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    if "WORLD_SIZE" in os.environ and args.gpus != world:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    global MULTI
    MULTI = world > 1 or os.environ.get("RG_BENCH_FORCE_DIST") == "1"
    wl, spec = resolve(args, world)
    if args.impl == "reference":
        run_reference(args, rank, world, wl, spec)
        return
    run_own(args, rank, world, local_rank, wl, spec)


if __name__ == "__main__":
    main()
