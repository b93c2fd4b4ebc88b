"""The scenario-sharded governor steps with the DEVICE kernels as each rank's local step,
world size 2 over gloo, both ranks on cuda:0 (gpurun gives one GPU; gloo runs the
collectives through the host, so no kernel waits on another rank's kernel).

This is the multi-rank code path of sharded.py exactly as it runs under NCCL on 8 GPUs --
the kernels write device-resident per-row counts / violation flags and the all-reduces run
on the library's stream -- except for the collective's transport.  Checked against the
real reference's 2^20-scenario goldens (tests/golden/c4_1m_step.npz, c4_1m_seq.npz) and
against the unsharded oracle on small cases.
"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"

CASES = [
    # (x0, v_prev, r, n_sim, j_star, m_grid, mag, seed, prefix)
    ([0.0, 0.0, 0.0], 0.0, 0.5, 64, 64, 16, 0.001, 7, False),
    ([0.1, 0.3, 0.05], 0.3, 2.4, 1001, 128, 32, 0.02, 11, False),
    ([0.1, 0.3, 0.05], 0.3, 2.4, 1001, 128, 32, 0.02, 11, True),
    ([2.0, 0.0, 0.0], 0.5, 0.6, 9, 32, 8, 0.001, 3, False),   # nothing feasible
    ([-0.3, -0.4, -0.1], -0.4, -0.4, 33, 64, 8, 0.01, 5, False),  # all rows duplicate
    ([0.05, 0.1, 0.02], 0.1, -2.5, 3000, 256, 32, 0.02, 19, False),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, big):
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2510_08288_b200 as rg
    from paper_2510_08288_b200 import sharded

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plant = rg.make_plant("surrogate-fc")
    box = rg.ConstraintSet(-0.9, 0.9, 0.0)
    out = {}
    if big:
        with np.load(GOLD / "c4_1m_step.npz") as z:
            g = {k: z[k] for k in z.files}
        n, js, m = int(g["n_sim"]), int(g["j_star"]), int(g["m_grid"])
        scen = rg.sample_scenarios(rg.DisturbanceModel.scaled(float(g["range"]), 3), n, js + 1,
                                   seed=int(g["seed"]))
        cfg = rg.GovernorConfig(j_star=js, m_grid=m, n_sim=n, n_kappa=8)
        a = sharded.robust_rg_parallel_sharded(plant, g["x0"], rg.GovernorState(float(g["v_prev"])),
                                               float(g["r"]), box, scen, cfg)
        b = sharded.robust_rg_sequential_sharded(plant, g["x0"],
                                                 rg.GovernorState(float(g["v_prev"])),
                                                 float(g["r"]), box, scen, cfg)
        c = sharded.robust_rg_joint_sharded(plant, g["x0"], rg.GovernorState(float(g["v_prev"])),
                                            float(g["r"]), box, scen, cfg)
        out["grid"] = [a.kappa_opt, a.v_applied, float(a.feasible)]
        out["words"] = a.diagnostics["row_words"]
        out["exch"] = a.diagnostics["device_exchange"]
        out["seq"] = [b.kappa_opt, b.v_applied, float(b.feasible), b.diagnostics["sims_run"],
                      b.diagnostics["early_terms"]]
        out["joint"] = [c.kappa_opt, c.v_applied, float(c.feasible)]
    else:
        res = []
        for (x0, vp, r, n, js, m, mag, seed, prefix) in CASES:
            model = rg.DisturbanceModel.scaled(mag, 3)
            scen = rg.sample_scenarios(model, n, js + 1, seed=seed)
            cfg = rg.GovernorConfig(j_star=js, m_grid=m, n_sim=n, prefix_mode=prefix)
            g = sharded.robust_rg_parallel_sharded(plant, np.array(x0), rg.GovernorState(vp), r,
                                                   box, scen, cfg)
            b = sharded.robust_rg_sequential_sharded(plant, np.array(x0), rg.GovernorState(vp),
                                                     r, box, scen, cfg)
            j = sharded.robust_rg_joint_sharded(plant, np.array(x0), rg.GovernorState(vp), r,
                                                box, scen, cfg)
            # the unsharded device calls on the same scenarios
            g1 = rg.robust_rg_parallel(plant, np.array(x0), rg.GovernorState(vp), r, box, scen,
                                       cfg)
            b1 = rg.robust_rg_sequential(plant, np.array(x0), rg.GovernorState(vp), r, box,
                                         scen, cfg)
            res.append([g.kappa_opt, g.v_applied, float(g.feasible), b.kappa_opt, b.v_applied,
                        float(b.feasible), b.diagnostics["sims_run"],
                        b.diagnostics["early_terms"], j.kappa_opt, j.v_applied,
                        float(j.feasible), g1.kappa_opt, b1.kappa_opt,
                        b1.diagnostics["sims_run"], b1.diagnostics["early_terms"]])
        out["cases"] = res
    np.save(Path(out_dir) / f"rank{rank}.npy", np.array([out], dtype=object), allow_pickle=True)
    dist.destroy_process_group()


def _run(tmp_path, big):
    import torch.multiprocessing as mp

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), big), nprocs=world,
                       join=True, start_method="spawn")
    r0 = np.load(tmp_path / "rank0.npy", allow_pickle=True)[0]
    r1 = np.load(tmp_path / "rank1.npy", allow_pickle=True)[0]
    return r0, r1


def test_sharded_device_steps_small_cases(tmp_path, orc):
    r0, r1 = _run(tmp_path, False)
    assert r0 == r1 or all(np.array_equal(a, b) for a, b in zip(r0["cases"], r1["cases"]))
    tlo, thi = orc.tighten(-0.9, 0.9, 0.0, 0.05)
    for i, (x0, vp, r, n, js, m, mag, seed, prefix) in enumerate(CASES):
        got = r0["cases"][i]
        d = orc.sample(seed, n, js + 1, [(-mag, mag)] * 3)
        kg, vg, fg, _, _, _ = orc.grid_step(0.01, np.array(x0), vp, r, m, d, -0.9, 0.9, tlo,
                                            thi, js, prefix_mode=prefix)
        kb, vb, fb, cells, early, _ = orc.robust_sequential(0.01, np.array(x0), vp, r, -0.9,
                                                            0.9, tlo, thi, d, js, 8)
        kj, fj, _ = orc.joint_bisect(0.01, np.array(x0), vp, r, -0.9, 0.9, tlo, thi, d, js, 8)
        assert got[:3] == [kg, vg, float(fg)], (i, got[:3])
        assert got[3:8] == [kb, vb, float(fb), cells, early], (i, got[3:8])
        assert got[8] == kj and got[10] == float(fj), i
        # the unsharded device calls agree with the sharded ones
        assert got[11] == got[0] and got[12:15] == [got[3], got[6], got[7]], i


def test_sharded_device_steps_at_2_20_scenarios_match_reference(tmp_path):
    """C4's 2^20-scenario step sharded over two ranks: the grid decision, the per-row
    verdicts, and Alg. 2's kappa / v / feasible / rollouts / early terminations equal the
    real reference's (multicore fill and robust_rg_sequential in the build container)."""
    r0, r1 = _run(tmp_path, True)
    for k in ("grid", "seq", "joint", "words"):
        assert r0[k] == r1[k], k
    with np.load(GOLD / "c4_1m_step.npz") as z:
        g = {k: z[k] for k in z.files}
    with np.load(GOLD / "c4_1m_seq.npz") as z:
        seq = [float(v) for v in z["result"]]
    assert r0["exch"], "the device-resident exchange path must run"
    assert r0["grid"] == [float(v) for v in g["result"]]
    n = int(g["n_sim"])
    words = np.array(r0["words"])
    counts = g["row_counts"]
    # gated rows (count 0 in the reference's P with a -1 word), feasible rows (word 0),
    # and violated rows (word > 0) -- the reference's P row sums say which is which
    feasible = counts == n
    assert np.array_equal(words == 0, feasible)
    assert np.all(words[~feasible] != 0)
    assert r0["seq"] == seq
    assert r0["joint"][0] == seq[0] and r0["joint"][2] == seq[2]
