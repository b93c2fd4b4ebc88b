"""The fused cross-GPU exchange of the scenario-sharded grid step (rg_xchg_*, RG_XCHG).

gpurun has one GPU, so the exchange runs with one rank (its window mapped once): the
kernel's whole protocol -- stores into every rank's window, the epoch flag, the wait, the
MAX over ranks and the extraction -- runs, and its result must equal the unexchanged step
bit for bit.  A second rank that never arrives is injected to check that the step fails
loudly after the timeout instead of hanging.  (Running two ranks whose kernels wait on
each other on one GPU is not done: see B200_PROFILING.md.)
"""

from __future__ import annotations

import os
import socket
import sys
import time
from pathlib import Path

import numpy as np
import pytest

import paper_2510_08288_b200 as rg
from paper_2510_08288_b200 import _capi

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _problem(j_star):
    tight = rg.tighten(rg.ConstraintSet(-0.9, 0.9, 0.0), 0.05)
    lo, hi = rg.admissible_setpoints(tight.lower, tight.upper)
    return _capi.Problem(0.01, -0.9, 0.9, lo, hi, j_star, 0)


@pytest.fixture
def xctx():
    ctx = _capi.context(0)
    ctx.xchg_connect(ctx.xchg_init(0, 1))
    yield ctx
    ctx.xchg_close()


def test_exchanged_step_equals_plain_step(xctx):
    rng = np.random.default_rng(12)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    for trial in range(24):
        n = int(rng.choice([1, 37, 1000, 3000, 20000]))
        M = int(rng.choice([2, 8, 32, 64]))
        js = int(rng.choice([16, 128]))
        prob = _problem(js)
        vp = float(rng.uniform(-1.2, 1.2))
        r = float(rng.uniform(-3, 3)) if trial % 5 else vp   # every 5th: all rows duplicate
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.06, 0.06, 3)
        sc = _capi.make_scenarios(500 + trial, 0, n, m.lo, m.span)
        prefix = bool(trial % 3 == 1)
        for abandon in (False, True):
            a = xctx.grid_step(prob, x0, vp, r, M, prefix, None, n, sc, not abandon,
                               abandon=abandon)
            b = xctx.grid_step(prob, x0, vp, r, M, prefix, None, n, sc, not abandon,
                               abandon=abandon, xchg=True)
            assert a[0].row == b[0].row, (trial, abandon)
            assert (a[0].sims_run, a[0].ss_pruned_rows, a[0].dedup_rows) == \
                (b[0].sims_run, b[0].ss_pruned_rows, b[0].dedup_rows)
            if not abandon:
                assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]), trial
                assert (a[0].early_terms, a[0].overflows) == (b[0].early_terms, b[0].overflows)
            else:  # abandoned counts differ run to run; the verdict words agree on zero
                assert np.array_equal(a[1] == 0, b[1] == 0)


def test_missing_peer_fails_loudly_not_hangs():
    """A second 'rank' that never runs (its window is our own, so its flag never rises):
    the step gives up after xchg_timeout_ms with RefgovError, and the context works on."""
    ctx = _capi.context(0)
    h = ctx.xchg_init(0, 2)
    ctx.xchg_connect(h + h)
    ctx.set_option("xchg_timeout_ms", 300)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    sc = _capi.make_scenarios(9, 0, 500, m.lo, m.span)
    t0 = time.perf_counter()
    try:
        with pytest.raises(rg.RefgovError, match="did not arrive"):
            ctx.grid_step(_problem(32), np.zeros(3), 0.0, 0.5, 16, False, None, 500, sc, False,
                          xchg=True)
        assert time.perf_counter() - t0 < 30
    finally:
        ctx.set_option("xchg_timeout_ms", 10000)
        ctx.xchg_close()
    res, viol, _ = ctx.grid_step(_problem(32), np.zeros(3), 0.0, 0.5, 16, False, None, 500, sc,
                                 False)
    assert res.row == 15


def test_fused_joint_search_equals_local_search(xctx):
    """rg_bisect_joint_sharded with one rank (the per-round exchange through its window)
    against the local persistent search and the per-iteration form: kappa, found, cells."""
    rng = np.random.default_rng(33)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    for trial in range(30):
        n = int(rng.choice([1, 100, 1000, 4000]))
        prob = _problem(int(rng.choice([16, 128, 256])))
        vp = float(rng.uniform(-1.2, 1.2))
        r = float(rng.uniform(-3, 3))
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.06, 0.06, 3)
        sc = _capi.make_scenarios(800 + trial, 0, n, m.lo, m.span)
        nk = int(rng.choice([1, 8, 12]))
        a = xctx.bisect_joint(prob, x0, vp, r, nk, None, n, sc)
        b = xctx.bisect_joint_sharded(prob, x0, vp, r, nk, None, n, sc, n)
        c = xctx.bisect_joint(prob, x0, vp, r, nk, None, n, sc, per_iteration=True)
        assert (a.kappa, a.found, a.cells) == (b.kappa, b.found, b.cells) == \
            (c.kappa, c.found, c.cells), trial
    # a grid step and a search interleave on one epoch sequence
    sc = _capi.make_scenarios(1, 0, 2000, m.lo, m.span)
    g = xctx.grid_step(_problem(64), np.zeros(3), 0.0, 0.5, 32, False, None, 2000, sc, False,
                       xchg=True)
    b = xctx.bisect_joint_sharded(_problem(64), np.zeros(3), 0.0, 2.5, 8, None, 2000, sc, 2000)
    g2 = xctx.grid_step(_problem(64), np.zeros(3), 0.0, 0.5, 32, False, None, 2000, sc, False,
                        xchg=True)
    assert g[0].row == g2[0].row == 31 and b.found


def test_fused_joint_search_missing_peer_fails_loudly():
    ctx = _capi.context(0)
    h = ctx.xchg_init(0, 2)
    ctx.xchg_connect(h + h)
    ctx.set_option("xchg_timeout_ms", 300)
    m = rg.DisturbanceModel.scaled(0.02, 3)
    sc = _capi.make_scenarios(9, 0, 500, m.lo, m.span)
    try:
        with pytest.raises(rg.RefgovError, match="did not arrive"):
            ctx.bisect_joint_sharded(_problem(32), np.zeros(3), 0.0, 2.5, 8, None, 500, sc, 500)
    finally:
        ctx.set_option("xchg_timeout_ms", 10000)
        ctx.xchg_close()
    r = ctx.bisect_joint(_problem(32), np.zeros(3), 0.0, 2.5, 8, None, 500, sc)
    assert r.found


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_2510_08288_b200 import sharded

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plant = rg.make_plant("surrogate-fc")
    box = rg.ConstraintSet(-0.9, 0.9, 0.0)
    rng = np.random.default_rng(4)
    res = []
    for trial in range(10):
        vp = float(rng.uniform(-1, 1))
        r = float(rng.uniform(-2.5, 2.5))
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.05, 0.05, 3)
        scen = rg.sample_scenarios(rg.DisturbanceModel.scaled(0.02, 3), 4000, 129, seed=70 + trial)
        cfg = rg.GovernorConfig(j_star=128, m_grid=32, n_sim=4000, prefix_mode=trial % 2 == 1)
        out = []
        for ex in ("nccl", "p2p"):
            k = sharded.robust_rg_parallel_sharded(plant, x0, rg.GovernorState(vp), r, box, scen,
                                                   cfg, exchange=ex)
            out.append((k.kappa_opt, k.v_applied, k.feasible,
                        [w == 0 for w in k.diagnostics["row_words"]]))
        res.append(out[0] == out[1])
        jt = [sharded.robust_rg_joint_sharded(plant, x0, rg.GovernorState(vp), r, box, scen, cfg,
                                              exchange=ex) for ex in ("nccl", "p2p")]
        res.append((jt[0].kappa_opt, jt[0].feasible, jt[0].diagnostics["sims_run"]) ==
                   (jt[1].kappa_opt, jt[1].feasible, jt[1].diagnostics["sims_run"]))
        res.append(jt[1].diagnostics.get("exchange") == "p2p")
    np.save(Path(out_dir) / "xchg.npy", np.array(res))
    dist.destroy_process_group()


def test_sharded_step_p2p_exchange_equals_collective(tmp_path):
    """robust_rg_parallel_sharded(exchange="p2p") against the collective exchange, one rank
    (its window set up through the same all_gather_object of IPC handles as with N)."""
    import torch.multiprocessing as mp

    mp.start_processes(_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True,
                       start_method="spawn")
    assert np.load(tmp_path / "xchg.npy").all()
