"""The B200 library plugged into the UNMODIFIED reference package (refgov_plugin.install).

The reference is the copy oracle/Makefile stages into oracle/_ref (it travels to the GPU
box; /root/reference does not).  CPU tests check the registration itself; the -m gpu
tests drive the reference's own entry points, harness, FastAPI service and click CLI with
backend "cuda" (and the in-process "gpu" seam) and compare with its CPU backends.
"""

from __future__ import annotations

import asyncio

import numpy as np
import pytest

from oracle import reference

refgov, _why = reference.load()
pytestmark = pytest.mark.skipif(refgov is None, reason=f"reference not staged: {_why}")

from paper_2510_08288_b200 import refgov_plugin  # noqa: E402


@pytest.fixture
def plugged():
    refgov_plugin.install(refgov)
    yield refgov
    refgov_plugin.uninstall(refgov)


def _call(app, method, path, payload=None):
    import httpx

    async def go():
        transport = httpx.ASGITransport(app=app)
        async with httpx.AsyncClient(transport=transport, base_url="http://svc") as client:
            return await client.request(method, path, json=payload)

    return asyncio.run(go())


def test_install_registers_backend_and_uninstall_restores():
    before = refgov.governor.BACKENDS
    fill0 = refgov.governor.fill_feasibility
    refgov_plugin.install(refgov)
    refgov_plugin.install(refgov)  # idempotent
    assert refgov.governor.BACKENDS == tuple(before) + ("cuda",)
    cfg = refgov.GovernorConfig(backend="cuda")  # the reference's own validation accepts it
    assert cfg.backend == "cuda"
    assert refgov.load_config({"governor": {"backend": "cuda"}}).governor.backend == "cuda"
    refgov_plugin.uninstall(refgov)
    assert refgov.governor.BACKENDS == before and refgov.governor.fill_feasibility is fill0
    with pytest.raises(refgov.ConfigError):
        refgov.GovernorConfig(backend="cuda")


def test_other_backends_untouched(plugged):
    plant = plugged.make_plant("surrogate-fc")
    box = plugged.ConstraintSet(-0.9, 0.9)
    scen = plugged.sample_scenarios(plugged.DisturbanceModel.scaled(0.02, 3), 16, 33, seed=3)
    cfg = plugged.GovernorConfig(j_star=32, n_sim=16, m_grid=8, backend="serial")
    a = plugged.robust_rg_parallel(plant, np.zeros(3), plugged.GovernorState(0.0), 1.5, box, scen,
                                   cfg)
    assert a.diagnostics["backend"] == "serial"


@pytest.mark.gpu
def test_reference_entry_points_on_the_device(plugged):
    """robust_rg_parallel / fill_feasibility / run_closed_loop of the stock reference with
    backend "cuda" equal its multicore backend bit for bit (P, decision, stats)."""
    rf = plugged
    plant = rf.make_plant("surrogate-fc")
    box = rf.ConstraintSet(-0.9, 0.9, anchor=0.0)
    model = rf.DisturbanceModel.scaled(0.02, 3)
    rng = np.random.default_rng(8)
    for trial in range(8):
        vp = float(rng.uniform(-1, 1))
        r = float(rng.uniform(-2.5, 2.5))
        x0 = np.array([np.tanh(vp), vp, np.tanh(vp) / 2]) + rng.uniform(-0.05, 0.05, 3)
        scen = rf.sample_scenarios(model, 500, 257, seed=600 + trial)
        out = {}
        for be in ("cuda", "multicore"):
            cfg = rf.GovernorConfig(j_star=256, n_sim=500, m_grid=32, backend=be)
            out[be] = rf.robust_rg_parallel(plant, x0, rf.GovernorState(vp), r, box, scen, cfg)
        a, b = out["cuda"], out["multicore"]
        assert np.array_equal(a.matrix, b.matrix), trial
        assert (a.kappa_opt, a.v_applied, a.feasible) == (b.kappa_opt, b.v_applied, b.feasible)
        for k in ("sims_run", "early_terms", "overflows", "ss_pruned_rows", "dedup_rows"):
            assert a.diagnostics[k] == b.diagnostics[k], (trial, k)
        assert a.diagnostics["backend"] == "cuda"
    setup = rf.load_config({"governor": {"n_sim": 64}, "steps": 300})
    runs = {}
    for be in ("cuda", "multicore"):
        g = rf.GovernorConfig(**{**setup.governor.__dict__, "backend": be})
        runs[be] = rf.run_closed_loop(setup.plant, setup.cset, setup.model, g, setup.profile,
                                      300, setup.seed)
    assert [r_[:6] for r_ in runs["cuda"].rows] == [r_[:6] for r_ in runs["multicore"].rows]


@pytest.mark.gpu
def test_reference_gpu_seam_in_process(plugged):
    """The stock "gpu" backend now reaches the device in process: P equals the multicore
    fill of the float32-rounded scenarios its protocol carries (backend_gpu.py:82)."""
    rf = plugged
    assert rf.backend_gpu.available()
    plant = rf.make_plant("surrogate-fc")
    box = rf.ConstraintSet(-0.9, 0.9)
    scen = rf.sample_scenarios(rf.DisturbanceModel.scaled(0.02, 3), 300, 129, seed=91)
    x0 = np.array([0.2, 0.35, 0.1])
    grid = rf.grid_kappas(32)
    st: dict = {}
    P = rf.fill_feasibility("gpu", plant, x0, 0.3, 2.3, grid, scen, box, 0.05, 128, stats=st)
    ref = rf.fill_feasibility("multicore", plant, x0, 0.3, 2.3, grid,
                              rf.ScenarioSet(scen.data.astype(np.float32).astype(np.float64)),
                              box, 0.05, 128)
    assert np.array_equal(P, ref)
    assert st["backend"] == "gpu" and st["sims_run"] == 32 * 300


@pytest.mark.gpu
def test_reference_service_cli_and_bench_on_the_device(plugged, tmp_path):
    """The reference's FastAPI service (/health, /govern/step, /bench), its click CLI
    (`refgov bench --backends cuda,gpu`, in-process ASGI) and bench_sweep run on the device."""
    rf = plugged
    from click.testing import CliRunner
    from refgov.cli import cli
    from refgov.service.app import create_app

    app = create_app()
    health = _call(app, "GET", "/health").json()
    assert health["backends"]["gpu"] is True
    cfg = {"governor": {"j_star": 64, "n_sim": 200, "m_grid": 16, "backend": "cuda"}}
    body = _call(app, "POST", "/govern/step", {"config": cfg, "r": 2.5, "v_prev": 0.0,
                                                "t": 3}).json()
    setup = rf.load_config(cfg)
    g = setup.governor
    scen = rf.sample_scenarios(setup.model, g.n_sim, g.j_star + 1,
                               seed=rf.derive_seed(setup.seed, "scenarios") + 3)
    direct = rf.robust_rg_parallel(setup.plant, np.zeros(3), rf.GovernorState(0.0), 2.5,
                                   setup.cset, scen, rf.GovernorConfig(
                                       **{**g.__dict__, "backend": "multicore"}))
    assert (body["kappa_opt"], body["v_applied"], body["feasible"]) == \
        (direct.kappa_opt, direct.v_applied, direct.feasible)
    assert body["diagnostics"]["backend"] == "cuda"
    bench = _call(app, "POST", "/bench", {"config": cfg, "n_sim": [64, 256],
                                          "backends": ["cuda", "gpu"], "reps": 2,
                                          "modes": ["kernel-only"]}).json()
    assert bench["skipped"] == 0 and len(bench["records"]) == 4
    out = tmp_path / "timing.csv"
    res = CliRunner().invoke(cli, ["bench", "--backends", "cuda,gpu", "--nsim", "64", "--reps",
                                   "2", "--modes", "kernel-only", "--out", str(out)])
    assert res.exit_code == 0, res.output
    lines = out.read_text().splitlines()
    assert lines[0] == "backend,n_sim,mode,mean_us,min_us,max_us,reps"
    assert {ln.split(",")[0] for ln in lines[1:]} == {"cuda", "gpu"}
