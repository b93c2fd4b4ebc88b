"""Multi-rank host logic of the sharded governor steps, world size 2 over gloo (CPU).

The device kernel is replaced by the CPU oracle as each rank's local step; the
sharding, the all-reduces and the extraction are the product code
(paper_2510_08288_b200/sharded.py).  Results must equal the unsharded oracle.
"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]

CASES = [
    # (x0, v_prev, r, n_sim, j_star, m_grid, mag, seed, prefix)
    ([0.0, 0.0, 0.0], 0.0, 0.5, 64, 64, 16, 0.001, 7, False),
    ([0.1, 0.3, 0.05], 0.3, 2.4, 101, 128, 32, 0.02, 11, False),
    ([0.1, 0.3, 0.05], 0.3, 2.4, 101, 128, 32, 0.02, 11, True),
    ([2.0, 0.0, 0.0], 0.5, 0.6, 9, 32, 8, 0.001, 3, False),   # nothing feasible
    ([-0.3, -0.4, -0.1], -0.4, -0.4, 33, 64, 8, 0.01, 5, False),  # all rows duplicate
]


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
    import torch.distributed as dist

    import paper_2510_08288_b200 as rg
    from oracle import oracle as orc
    from paper_2510_08288_b200 import sharded

    dist.init_process_group("gloo", rank=rank, world_size=world)
    plant = rg.make_plant("surrogate-fc")
    box = rg.ConstraintSet(-0.9, 0.9)
    tlo, thi = orc.tighten(-0.9, 0.9, 0.0, 0.05)
    results = []
    for (x0, vp, r, n, js, m, mag, seed, prefix) in CASES:
        model = rg.DisturbanceModel.scaled(mag, 3)
        scen = rg.sample_scenarios(model, n, js + 1, seed=seed)
        cfg = rg.GovernorConfig(j_star=js, m_grid=m, n_sim=n, prefix_mode=prefix)

        def grid_local(shard):
            d = orc.sample(shard.seed, shard.n_sim, shard.horizon, model.ranges, k0=shard.k0)
            P, S, _, _ = orc.fill_feasibility(0.01, np.array(x0), vp, r, orc.grid_kappas(m), d,
                                              -0.9, 0.9, tlo, thi, js)
            grid = orc.grid_kappas(m)
            ok = np.array([orc.ss_ok(orc.update_setpoint(vp, r, float(k)), tlo, thi)
                           for k in grid])
            return np.where(ok, (~P).sum(axis=1), sharded.PRUNED).astype(np.uint32)

        def bis_local(shard):
            d = orc.sample(shard.seed, shard.n_sim, shard.horizon, model.ranges, k0=shard.k0)
            k, _, f, cells, early, _ = orc.robust_sequential(0.01, np.array(x0), vp, r, -0.9,
                                                             0.9, tlo, thi, d, js, 8)
            return k, int(f), cells, early

        class OracleJointShard:
            """Rank-local joint iterations on the CPU oracle (same methods as the device)."""

            def begin(self, prob, x0_, v_prev, r_, n_kappa, dist_t, n_sim, stream):
                self.d = orc.sample(stream.seed, stream.n_sim, js + 1, model.ranges,
                                    k0=stream.k0)
                self.lo, self.hi, self.kopt, self.found, self.done = 0.0, 1.0, 0.0, False, False
                self.cells = self.early = 0
                self.n_kappa = n_kappa
                import torch
                self._flag = torch.zeros(1, dtype=torch.int32)

            def _kappa(self, it):
                return 1.0 if it < 0 else 0.5 * (self.lo + self.hi)

            def roll(self, it):
                self._flag.zero_()
                if self.done:
                    return
                v = orc.update_setpoint(vp, r, self._kappa(it))
                if not orc.ss_ok(v, tlo, thi):
                    return
                for k in range(self.d.shape[0]):
                    st, _ = orc.cell_sfc(0.01, np.array(x0), v, self.d[k], js, -0.9, 0.9)
                    if st != orc.CELL_OK:
                        self._flag[0] = 1
                        break

            def flag(self):
                return self._flag

            def stream(self):
                return None

            def decide(self, it):
                if self.done:
                    return
                kappa = self._kappa(it)
                v = orc.update_setpoint(vp, r, kappa)
                feas = orc.ss_ok(v, tlo, thi) and int(self._flag[0]) == 0
                if it < 0:
                    if feas:
                        self.kopt, self.found, self.done = 1.0, True, True
                elif feas:
                    self.kopt, self.found, self.lo = kappa, True, kappa
                else:
                    self.hi = kappa
                if it == self.n_kappa - 1:
                    self.done = True

            def end(self):
                return self.kopt, self.found, self.cells, self.early

        jr = sharded.robust_rg_joint_sharded(plant, np.array(x0), rg.GovernorState(vp), r, box,
                                             scen, cfg, shard_impl=OracleJointShard())
        g = sharded.robust_rg_parallel_sharded(plant, np.array(x0), rg.GovernorState(vp), r,
                                               box, scen, cfg, local_step=grid_local)
        b = sharded.robust_rg_sequential_sharded(plant, np.array(x0), rg.GovernorState(vp), r,
                                                 box, scen, cfg, local_step=bis_local)
        results.append([g.kappa_opt, g.v_applied, float(g.feasible), b.kappa_opt, b.v_applied,
                        float(b.feasible), b.diagnostics["sims_run"],
                        b.diagnostics["early_terms"], jr.kappa_opt, jr.v_applied,
                        float(jr.feasible)])
    np.save(Path(out_dir) / f"rank{rank}.npy", np.array(results))
    dist.destroy_process_group()


def test_sharded_steps_equal_unsharded_oracle(tmp_path, orc):
    import torch.multiprocessing as mp

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    r0 = np.load(tmp_path / "rank0.npy")
    r1 = np.load(tmp_path / "rank1.npy")
    assert np.array_equal(r0, r1), "ranks disagree"
    tlo, thi = orc.tighten(-0.9, 0.9, 0.0, 0.05)
    for i, (x0, vp, r, n, js, m, mag, seed, prefix) in enumerate(CASES):
        d = orc.sample(seed, n, js + 1, [(-mag, mag)] * 3)
        kg, vg, fg, _, _, _ = orc.grid_step(0.01, np.array(x0), vp, r, m, d, -0.9, 0.9, tlo,
                                            thi, js, prefix_mode=prefix)
        kb, vb, fb, cells, early, _ = orc.robust_sequential(0.01, np.array(x0), vp, r, -0.9,
                                                            0.9, tlo, thi, d, js, 8)
        kj, fj, _ = orc.joint_bisect(0.01, np.array(x0), vp, r, -0.9, 0.9, tlo, thi, d, js, 8)
        vj = orc.update_setpoint(vp, r, kj)
        expect = [kg, vg, float(fg), kb, vb, float(fb), cells, early, kj, vj, float(fj)]
        assert list(r0[i]) == expect, (i, list(r0[i]), expect)
        # the joint search lands where the per-scenario bisections' minimum does
        assert (kj, fj) == (kb, fb), (i, kj, fj, kb, fb)


def test_extract_row_matches_reference_extraction():
    from paper_2510_08288_b200 import extract_kappa_opt
    from paper_2510_08288_b200.sharded import extract_row

    rng = np.random.default_rng(0)
    for _ in range(500):
        m = int(rng.integers(2, 12))
        counts = rng.integers(0, 3, m) * rng.integers(0, 2, m)
        dup = np.full(m, -1)
        P = np.stack([np.full(4, c == 0) for c in counts])
        for prefix in (False, True):
            row, _ = extract_kappa_opt(P, prefix_mode=prefix)
            got = extract_row(counts.astype(np.int64), dup, prefix)
            assert (None if row is None else row - 1) == got


def _worker_empty(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    import paper_2510_08288_b200 as rg
    from paper_2510_08288_b200 import sharded

    dist.init_process_group("gloo", rank=rank, world_size=world)
    plant = rg.make_plant("surrogate-fc")
    box = rg.ConstraintSet(-0.9, 0.9)
    scen = rg.sample_scenarios(rg.DisturbanceModel.scaled(0.01, 3), 1, 33, seed=1)
    cfg = rg.GovernorConfig(j_star=32, m_grid=8, n_sim=1)
    raised = []
    for fn in (sharded.robust_rg_parallel_sharded, sharded.robust_rg_sequential_sharded,
               sharded.robust_rg_joint_sharded):
        try:
            fn(plant, np.zeros(3), rg.GovernorState(0.0), 0.5, box, scen, cfg,
               **({"local_step": lambda sh: None} if fn is not sharded.robust_rg_joint_sharded
                  else {"shard_impl": object()}))
        except rg.ConfigError:
            raised.append(1)
    dist.barrier()  # every rank got here: nobody was left waiting in a collective
    np.save(Path(out_dir) / f"empty{rank}.npy", np.array(raised))
    dist.destroy_process_group()


def test_empty_shards_rejected_on_every_rank(tmp_path):
    """n_sim < world: every rank raises ConfigError before any collective."""
    import torch.multiprocessing as mp

    mp.start_processes(_worker_empty, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    for r in (0, 1):
        assert np.load(tmp_path / f"empty{r}.npy").tolist() == [1, 1, 1]
