"""Register the B200 library as a backend of an unmodified ``refgov`` package.

The reference selects where its feasibility matrix is filled by a backend name
(``BACKENDS = ("serial", "multicore", "gpu")``, governor.py:53) and dispatches on it
inside ``fill_feasibility`` (governor.py:245-348); its "gpu" backend reaches a device
through ``backend_gpu.fill`` (backend_gpu.py:50-140: a subprocess and temp files).
``install()`` plugs this library into both seams of a live ``refgov`` module, so the
reference's own entry points, harness, FastAPI service and CLI run on the B200:

* backend ``"cuda"`` is appended to ``BACKENDS`` and ``fill_feasibility`` gains a
  ``"cuda"`` branch that runs this package's device fill (``rg_fill`` through the C ABI,
  with the reference's host gate / dedup / stats semantics, governor.py:286-347);
* with ``gpu_seam=True`` (default) ``backend_gpu.fill`` / ``available`` are replaced by an
  in-process device fill with the same contract (P and the runner's stats keys), so the
  stock ``"gpu"`` backend, ``GET /health`` (``"gpu": true``) and ``refgov bench --backends
  gpu`` reach the device without ``REFGOV_GPU_RUNNER``.

Nothing else of the reference changes: its grid extraction, bisection drivers, closed
loop, config validation and error mapping run as shipped.  This is INTEGRATION.md §B's
``backend_cuda.py`` as a runtime plugin instead of a file added to the reference.
"""

from __future__ import annotations

import time

import numpy as np

__all__ = ["install", "uninstall"]

_SAVED = "__b200_plugin_saved__"


def install(refgov=None, device: int = 0, gpu_seam: bool = True):
    """Plug the device into ``refgov`` (imported if not given); returns the module.

    Idempotent.  ``uninstall(refgov)`` restores the original functions.
    """
    if refgov is None:
        import refgov  # noqa: F811  (the reference package on sys.path)
    G = refgov.governor
    BG = _backend_gpu(refgov)
    if getattr(G, _SAVED, None) is None:
        saved = {"BACKENDS": G.BACKENDS, "fill_feasibility": G.fill_feasibility,
                 "bg_fill": BG.fill, "bg_available": BG.available}
        setattr(G, _SAVED, saved)
    saved = getattr(G, _SAVED)
    orig_fill = saved["fill_feasibility"]

    def fill_feasibility(backend, plant, x0, v_prev, r_t, grid, scenarios, cset, eps, j_star,
                         workers=None, stats=None, tighten_mode="scale"):
        if backend != "cuda":
            return orig_fill(backend, plant, x0, v_prev, r_t, grid, scenarios, cset, eps,
                             j_star, workers=workers, stats=stats, tighten_mode=tighten_mode)
        from . import governor as dev

        st: dict = {}
        P = dev.fill_feasibility("cuda", plant, x0, v_prev, r_t, grid, scenarios, cset, eps,
                                 j_star, stats=st, tighten_mode=tighten_mode, device=device)
        if stats is not None:
            stats.update(st)
        return P

    fill_feasibility.__doc__ = orig_fill.__doc__
    G.BACKENDS = tuple(saved["BACKENDS"]) + ("cuda",)
    G.fill_feasibility = fill_feasibility
    refgov.fill_feasibility = fill_feasibility
    if gpu_seam:
        BG.fill = _device_fill_factory(device)
        BG.available = _available
    return refgov


def _backend_gpu(refgov):
    import importlib

    return importlib.import_module(refgov.__name__ + ".backend_gpu")


def uninstall(refgov) -> None:
    """Restore the functions ``install`` replaced."""
    G = refgov.governor
    saved = getattr(G, _SAVED, None)
    if saved is None:
        return
    G.BACKENDS = saved["BACKENDS"]
    G.fill_feasibility = saved["fill_feasibility"]
    refgov.fill_feasibility = saved["fill_feasibility"]
    BG = _backend_gpu(refgov)
    BG.fill = saved["bg_fill"]
    BG.available = saved["bg_available"]
    setattr(G, _SAVED, None)


def _available() -> bool:
    """backend_gpu.available (backend_gpu.py:45-47): a usable B200 and library."""
    from . import _capi
    from .errors import BackendUnavailableError

    try:
        return _capi.device_count() > 0 and _capi.context(0) is not None
    except BackendUnavailableError:
        return False


def _device_fill_factory(device: int):
    def fill(plant, x0, v_rows, dist, j_star, cset, tight):
        """backend_gpu.fill's contract in process (backend_gpu.py:50-140): the scenarios
        rounded to the float32 the protocol carries (write_rgsc, disturbance.py:216-226),
        every gated row rolled out on the device (the runner does not dedup), P = OK &
        steady-state gate, stats {kernel_us, total_us, sims_run, early_terms}."""
        from .errors import BackendUnavailableError
        from .runner import fill_rows

        if getattr(plant, "kernel_kind", None) != "surrogate-fc":  # backend_gpu.py:66-71
            raise BackendUnavailableError(
                "the device kernel is specialized to the surrogate plant; got plant kernel "
                f"kind {getattr(plant, 'kernel_kind', None)!r}")
        t0 = time.perf_counter()
        dist32 = np.asarray(dist, dtype=np.float32).astype(np.float64)
        P, early, kernel_us = fill_rows(plant.step_size, x0, v_rows, dist32, j_star,
                                        float(cset.lower), float(cset.upper),
                                        float(tight.lower), float(tight.upper), device)
        return P, {"kernel_us": kernel_us, "total_us": int((time.perf_counter() - t0) * 1e6),
                   "sims_run": int(np.size(v_rows) * dist32.shape[0]), "early_terms": early}

    return fill
