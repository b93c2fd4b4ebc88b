"""Scenario-sharded governor steps across GPUs.

One process per GPU (torchrun).  A generated ScenarioSet is split into
contiguous counter ranges, rank r simulating scenarios [k0 + r*n/W,
k0 + (r+1)*n/W) -- the counter RNG makes that free of scenario traffic
(disturbance.py:85-92).  The only exchange is per step:

* grid step (Alg. 3): the kernel writes this shard's per-row violating-scenario
  counts (int32, -1 for a gated-out row) into device memory and one all-reduce
  (MAX) runs on the library's stream right after it; a row is all-feasible iff
  its global count is 0, and every rank extracts the same row
  (extract_kappa_opt, governor.py:351-377).  128 bytes per step;
* exact Alg. 2: ONE all-reduce per step: every rank writes (kappa as its
  dyadic-number bits, found, cells, early) into its own slot of a zeroed
  int64[4 * world] vector and the SUM all-reduce gathers them; each rank then
  takes MIN kappa, AND found and the sums (governor.py:496-506);
* joint bisection: one all-reduce (MAX) of the uint32
  violation flag per iteration, enqueued on the library's stream between the
  local rollout kernel and the decision kernel, so the n_kappa + 1 iterations
  never wait on the host.

The collectives run through torch.distributed on device tensors: NCCL on the
GPUs, or gloo (which all-reduces CUDA tensors through the host) for the
world-size-2 tests that run both ranks on one GPU.  The local step is the
device kernel.
"""

from __future__ import annotations

import time

import numpy as np

from . import _capi
from .errors import ConfigError, InfeasibleError
from .governor import (KappaResult, _prepared, _source, _validate_state, _host_rows,
                       update_setpoint)
from .governor import _require_surrogate as _require_device_plant

__all__ = ["PRUNED", "global_row_counts", "extract_row", "robust_rg_parallel_sharded",
           "robust_rg_sequential_sharded", "combine_bisection", "robust_rg_joint_sharded",
           "DeviceJointShard"]

PRUNED = np.uint32(0xFFFFFFFF)  # rg_grid_step's marker for a gated-out row
_BIG = 1 << 40                  # > any scenario count; marks pruned rows in the sum


def _dist():
    import torch.distributed as dist

    return dist


def _check_shardable(scenarios, world: int) -> None:
    """Every rank needs at least one scenario.  The check reads only the global
    set, which every rank holds, so all ranks raise together before any device
    work or collective (no rank is left waiting in an all-reduce)."""
    if scenarios.n_sim < world:
        raise ConfigError(f"{scenarios.n_sim} scenarios cannot be sharded over {world} ranks "
                          "(each rank needs at least one)")


def global_row_counts(local_viol: np.ndarray, group=None, device=None) -> np.ndarray:
    """Sum per-row violation counts over ranks; pruned rows stay >= _BIG."""
    import torch

    c = np.where(local_viol == PRUNED, _BIG, local_viol.astype(np.int64))
    t = torch.as_tensor(c, dtype=torch.int64)
    if device is not None:
        t = t.to(device)
    _dist().all_reduce(t, op=_dist().ReduceOp.SUM, group=group)
    return t.cpu().numpy()


def extract_row(counts: np.ndarray, dup_src: np.ndarray, prefix_mode: bool) -> int | None:
    """0-based best all-feasible row from global counts (governor.py:351-377).

    Duplicate rows share their representative's verdict (governor.py:329-333).
    """
    src = np.where(dup_src >= 0, dup_src, np.arange(counts.size))
    full = counts[src] == 0
    if prefix_mode:
        bad = np.flatnonzero(~full)
        idx = (int(bad[0]) if bad.size else full.size) - 1
    else:
        ok = np.flatnonzero(full)
        idx = int(ok[-1]) if ok.size else -1
    return None if idx < 0 else idx


_DEV_COUNTS: dict = {}


def _device_row(ctx, dist, group, prob, x_t, v_prev, r_t, config, n_sim, stream):
    """The grid step with its exchange on the device: the kernel writes this shard's
    per-row counts (int32 view; a gated-out row is -1 on every rank) into a device
    buffer, one NCCL all-reduce (MAX) runs on the library's stream after it, and only
    the M reduced counts come back to the host.  The global MAX is 0 exactly for the
    rows feasible on every shard; duplicate rows already carry their source's count
    (the kernel's finalize), so the extraction needs no dedup map."""
    import torch

    key = (ctx.device, config.m_grid)
    viol = _DEV_COUNTS.get(key)
    if viol is None:
        viol = _DEV_COUNTS[key] = torch.empty(config.m_grid, dtype=torch.int32,
                                              device=f"cuda:{ctx.device}")
    ctx.grid_step_to_device(prob, x_t, v_prev, r_t, config.m_grid, config.prefix_mode, n_sim,
                            stream, viol.data_ptr())
    with torch.cuda.stream(torch.cuda.ExternalStream(ctx.stream_ptr,
                                                     device=f"cuda:{ctx.device}")):
        dist.all_reduce(viol, op=dist.ReduceOp.MAX, group=group)
        counts = viol.cpu().numpy()
    full = counts == 0
    if config.prefix_mode:
        bad = np.flatnonzero(~full)
        idx = (int(bad[0]) if bad.size else full.size) - 1
    else:
        ok = np.flatnonzero(full)
        idx = int(ok[-1]) if ok.size else -1
    return (None if idx < 0 else idx), counts


_P2P: dict = {}


def _p2p_ready(ctx, dist, group):
    """Map every rank's exchange window once per (device, group): rg_xchg_init, an
    all_gather_object of the CUDA IPC handles, rg_xchg_connect."""
    key = (ctx.device, id(group))
    if key not in _P2P:
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        mine = ctx.xchg_init(rank, world)
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        ctx.xchg_connect(b"".join(handles))
        _P2P[key] = True


def robust_rg_parallel_sharded(plant, x_t, state, r_t, cset, scenarios, config, group=None,
                               local_step=None, exchange="nccl"):
    """robust_rg_parallel over the ranks of `group`; every rank returns the same result.

    ``local_step(shard) -> uint32[M]`` computes this rank's per-row counts; the
    default is the device kernel (rg_grid_step) with the exchange on the device
    (_device_row).  A dense host scenario tensor is stepped synchronously and its
    counts all-reduced from the host.  matrix is None (P is sharded).

    ``exchange="p2p"`` (generated scenarios, m_grid <= 64, ranks on one node) fuses the
    exchange into the step kernel instead of an NCCL all-reduce: its finalizing block
    writes the shard's per-row words into every rank's window over NVLink and extracts
    the global row itself (rg_xchg_*, RG_XCHG).
    """
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    x_t = _validate_state(plant, x_t)
    _require_device_plant(plant)
    _check_shardable(scenarios, world)
    prob, interval, grid, grid_list = _prepared(plant.step_size, cset.lower, cset.upper,
                                                cset.anchor, config.epsilon,
                                                config.tighten_mode, config.j_star,
                                                config.m_grid)
    shard = scenarios.shard(rank, world)
    t0 = time.perf_counter()
    _, ss_ok, dup_src, rows = _host_rows(float(state.v_prev), float(r_t), grid_list, interval)
    ss_ok = np.array(ss_ok, dtype=bool)
    dup_src = np.array(dup_src, dtype=np.int64)
    counts = None
    if local_step is None:
        ctx = _capi.context(getattr(config, "device", 0))
        dist_t, n_sim, stream = _source(shard, config.j_star)
        if dist_t is None and exchange == "p2p":
            with ctx.lock:
                _p2p_ready(ctx, dist, group)
                res, viol, _ = ctx.grid_step(prob, x_t, state.v_prev, r_t, config.m_grid,
                                             config.prefix_mode, None, n_sim, stream, False,
                                             abandon=True, timing=False, xchg=True)
            counts = viol.view(np.int32)
            row = None if res.row < 0 else int(res.row)
        elif dist_t is None:
            with ctx.lock:
                row, counts = _device_row(ctx, dist, group, prob, x_t, state.v_prev, r_t,
                                          config, n_sim, stream)
        else:
            res, viol, _ = ctx.grid_step(prob, x_t, state.v_prev, r_t, config.m_grid,
                                         config.prefix_mode, dist_t, n_sim, stream, False,
                                         abandon=True)
            dev = f"cuda:{ctx.device}" if dist.get_backend(group) == "nccl" else None
            row = extract_row(global_row_counts(viol, group, dev), dup_src, config.prefix_mode)
    else:
        viol = np.asarray(local_step(shard), dtype=np.uint32)
        row = extract_row(global_row_counts(viol, group, None), dup_src, config.prefix_mode)
    diag = {"method": "parallel-grid-sharded", "ranks": world, "backend": "cuda",
            "device_exchange": counts is not None, "exchange": exchange,
            # global per-row verdict words: 0 = feasible on every shard, -1 = gated out,
            # > 0 = some shard violated (rows already known infeasible stop early, so a
            # positive word is not a full count)
            "row_words": None if counts is None else counts.tolist(),
            "sims_run": len(rows) * scenarios.n_sim,
            "ss_pruned_rows": int(np.count_nonzero(~ss_ok)),
            "dedup_rows": int(np.count_nonzero(dup_src >= 0)),
            "wall_us": int((time.perf_counter() - t0) * 1e6)}
    if row is None:
        if config.infeasible_policy == "error":
            raise InfeasibleError("no candidate feasible, including kappa=0 (hold current "
                                  "setpoint)")
        return KappaResult(0.0, state.v_prev, False, diag, None)
    kappa = float(grid[row])
    v = update_setpoint(state.v_prev, r_t, kappa)
    state.v_prev = v
    return KappaResult(kappa, v, True, diag, None)


def combine_bisection(kappa: float, found: int, cells: int, early: int, group=None,
                      device=None):
    """MIN kappa, AND found, SUM cells/early over ranks (governor.py:496-506), in ONE
    all-reduce: rank r writes (bits(kappa), found, cells, early) into slots 4r..4r+3 of a
    zeroed int64[4 * world] vector, the SUM all-reduce gathers every rank's four numbers,
    and each rank reduces them itself.  kappa >= 0, so its IEEE bits order like its
    value; the slots are exact (each is a sum of one number and zeros)."""
    import torch

    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    v = torch.zeros(4 * world, dtype=torch.int64)
    v[4 * rank: 4 * rank + 4] = torch.tensor(
        [int(np.float64(kappa).view(np.int64)), int(bool(found)), int(cells), int(early)],
        dtype=torch.int64)
    if device is not None:
        v = v.to(device)
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    a = v.cpu().numpy().reshape(world, 4)
    kappa = float(a[:, 0].min().astype(np.int64).view(np.float64))
    return kappa, bool(a[:, 1].min()), int(a[:, 2].sum()), int(a[:, 3].sum())


def robust_rg_sequential_sharded(plant, x_t, state, r_t, cset, scenarios, config, group=None,
                                 local_step=None):
    """robust_rg_sequential (exact Alg. 2) over the ranks of `group`.

    ``local_step(shard) -> (kappa, found, cells, early)`` defaults to rg_bisect.
    """
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    x_t = _validate_state(plant, x_t)
    _require_device_plant(plant)
    _check_shardable(scenarios, world)
    shard = scenarios.shard(rank, world)
    t0 = time.perf_counter()
    dev = None
    if local_step is None:
        prob, _, _, _ = _prepared(plant.step_size, cset.lower, cset.upper, cset.anchor,
                                  config.epsilon, config.tighten_mode, config.j_star, 0)
        ctx = _capi.context(getattr(config, "device", 0))
        dist_t, n_sim, stream = _source(shard, config.j_star)
        res, _, _ = ctx.bisect(prob, x_t, state.v_prev, r_t, config.n_kappa, dist_t, n_sim,
                               stream)
        local = (res.kappa, res.found, res.cells, res.early)
        dev = f"cuda:{ctx.device}"
    else:
        local = local_step(shard)
    kappa, found, cells, early = combine_bisection(*local, group=group, device=dev)
    v = update_setpoint(state.v_prev, r_t, kappa)
    state.v_prev = v
    return KappaResult(kappa, v, found, {"method": "sequential-sharded", "ranks": world,
                                         "sims_run": cells, "early_terms": early,
                                         "wall_us": int((time.perf_counter() - t0) * 1e6)})


class DeviceJointShard:
    """This rank's part of a joint bisection on its GPU (rg_joint_*).

    ``flag()`` is the device-resident uint32 violation flag as a torch tensor
    (no copy), and ``stream()`` the library's stream: the all-reduce between
    ``roll`` and ``decide`` runs there, in order with the kernels.
    """

    def __init__(self, ctx):
        self.ctx = ctx
        self._flag = None

    def begin(self, prob, x0, v_prev, r, n_kappa, dist, n_sim, scen):
        self.ctx.joint_begin(prob, x0, v_prev, r, n_kappa, dist, n_sim, scen)
        self._flag = None

    def roll(self, it):
        self.ctx.joint_iter(it, fold=False)

    def decide(self, it):
        self.ctx.joint_decide(it)

    def stream(self):
        import torch

        return torch.cuda.ExternalStream(self.ctx.stream_ptr, device=f"cuda:{self.ctx.device}")

    def flag(self):
        import torch

        if self._flag is None:
            ptr = self.ctx.joint_flag_ptr()

            class _Iface:  # __cuda_array_interface__ view of the flag word
                __cuda_array_interface__ = {"shape": (1,), "typestr": "<i4",
                                            "data": (ptr, False), "version": 3}

            self._flag = torch.as_tensor(_Iface(), device=f"cuda:{self.ctx.device}")
        return self._flag

    def end(self):
        res = self.ctx.joint_end()
        return float(res.kappa), bool(res.found), int(res.cells), int(res.early)


def robust_rg_joint_sharded(plant, x_t, state, r_t, cset, scenarios, config, group=None,
                            shard_impl=None, exchange="nccl"):
    """robust_rg_joint over the ranks of `group` (scenario shards, OR per iteration).

    ``shard_impl`` defaults to DeviceJointShard; the host-logic tests pass an
    oracle-backed object with the same methods.  Every rank walks the same
    candidates and returns the same kappa; sims_run / early_terms are summed.

    ``exchange="p2p"``: the whole search is one persistent kernel per GPU with the
    per-round OR of the shards' verdicts done inside it over NVLink
    (rg_bisect_joint_sharded), when the largest shard fits in one wave; otherwise, and
    for dense scenario tensors, the per-iteration form with a collective.
    """
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    x_t = _validate_state(plant, x_t)
    _require_device_plant(plant)
    _check_shardable(scenarios, world)
    shard = scenarios.shard(rank, world)
    prob, _, _, _ = _prepared(plant.step_size, cset.lower, cset.upper, cset.anchor,
                              config.epsilon, config.tighten_mode, config.j_star, 0)
    t0 = time.perf_counter()
    if exchange == "p2p" and shard_impl is None:
        got = _joint_p2p(dist, group, prob, x_t, state, r_t, config, scenarios, shard, world)
        if got is not None:
            kappa, found, cells, early, dev = got
            import torch
            ce = torch.tensor([cells, early], dtype=torch.int64, device=dev)
            dist.all_reduce(ce, op=dist.ReduceOp.SUM, group=group)
            cells, early = (int(x) for x in ce.cpu().tolist())
            v = update_setpoint(state.v_prev, r_t, kappa)
            state.v_prev = v
            return KappaResult(kappa, v, found, {"method": "joint-sharded", "ranks": world,
                                                 "exchange": "p2p", "sims_run": cells,
                                                 "early_terms": early,
                                                 "wall_us": int((time.perf_counter() - t0) * 1e6)})
    impl = shard_impl or DeviceJointShard(_capi.context(getattr(config, "device", 0)))
    lock = impl.ctx.lock if hasattr(impl, "ctx") else _nullcontext()
    with lock:  # begin .. end is one search on the context: no other call may interleave
        kappa, found, cells, early = _joint_iterations(impl, dist, group, prob, x_t, state, r_t,
                                                       config, shard)
    import torch

    ce = torch.tensor([cells, early], dtype=torch.int64)
    if hasattr(impl, "ctx"):
        ce = ce.to(f"cuda:{impl.ctx.device}")
    dist.all_reduce(ce, op=dist.ReduceOp.SUM, group=group)
    cells, early = (int(x) for x in ce.cpu().tolist())
    v = update_setpoint(state.v_prev, r_t, kappa)
    state.v_prev = v
    return KappaResult(kappa, v, found, {"method": "joint-sharded", "ranks": world,
                                         "sims_run": cells, "early_terms": early,
                                         "wall_us": int((time.perf_counter() - t0) * 1e6)})


def _joint_p2p(dist, group, prob, x_t, state, r_t, config, scenarios, shard, world):
    """The fused form, or None when it does not apply (every rank decides alike: the test
    reads only the global scenario count and kind)."""
    from .errors import ConfigError as _ConfigError

    ctx = _capi.context(getattr(config, "device", 0))
    dist_t, n_sim, stream = _source(shard, config.j_star)
    if dist_t is not None:
        return None
    n_max = -(-scenarios.n_sim // world)
    with ctx.lock:
        _p2p_ready(ctx, dist, group)
        try:
            res = ctx.bisect_joint_sharded(prob, x_t, state.v_prev, r_t, config.n_kappa, None,
                                           n_sim, stream, n_max)
        except _ConfigError:  # the largest shard exceeds one wave
            return None
    return float(res.kappa), bool(res.found), int(res.cells), int(res.early), \
        f"cuda:{ctx.device}"


def _joint_iterations(impl, dist, group, prob, x_t, state, r_t, config, shard):
    dist_t, n_sim, stream = _source(shard, config.j_star)
    impl.begin(prob, x_t, state.v_prev, r_t, config.n_kappa, dist_t, n_sim, stream)
    import torch

    st = impl.stream()
    cm = torch.cuda.stream(st) if st is not None else _nullcontext()
    with cm:
        for it in range(-1, config.n_kappa):
            impl.roll(it)
            dist.all_reduce(impl.flag(), op=dist.ReduceOp.MAX, group=group)
            impl.decide(it)
    return impl.end()


class _nullcontext:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False
