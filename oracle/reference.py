"""TEST INFRASTRUCTURE ONLY -- the unmodified reference package, for timing and checking.

``oracle/Makefile`` (target ``ref``, run by ``__graft_entry__.build()`` in the build
container) copies the reference's own Python package, ``/root/reference/pkg/src/refgov``,
into the git-ignored ``oracle/_ref/refgov``; gpurun ships it to the GPU box with the
working tree.  Its hot loop is numba-JIT FP64 (kernels.py:47-162), so it runs wherever
numba imports -- this image has numba 0.65.0.

Who may import this: bench.py's ``--impl reference`` arm and its ``cpu_baseline`` (the
timed CPU baseline), and tests (as a checker).  The product package never does.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

_HERE = Path(__file__).resolve().parent
REF_ROOT = _HERE / "_ref"

_mod = None
_why = None


def load():
    """(refgov module, None) or (None, reason).  Imports once; numba's JIT cache goes to
    NUMBA_CACHE_DIR (default /tmp/rg_numba_cache) so the read-only source tree is fine."""
    global _mod, _why
    if _mod is not None or _why is not None:
        return _mod, _why
    if not (REF_ROOT / "refgov" / "__init__.py").exists():
        _why = f"{REF_ROOT / 'refgov'} is not staged (run __graft_entry__.build() where " \
               "/root/reference exists)"
        return None, _why
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rg_numba_cache")
    try:
        import numba  # noqa: F401
    except Exception as e:  # pragma: no cover - image without numba
        _why = f"numba does not import: {e}"
        return None, _why
    if str(REF_ROOT) not in sys.path:
        sys.path.insert(0, str(REF_ROOT))
    try:
        import refgov
    except Exception as e:  # pragma: no cover
        _why = f"refgov does not import: {e}"
        return None, _why
    _mod = refgov
    return _mod, None


def threads() -> dict:
    """The host parallelism the reference's multicore backend uses (governor.py:241-242:
    workers=None -> os.cpu_count(); numba's pool has NUMBA_NUM_THREADS threads)."""
    import numba

    return {"os_cpu_count": os.cpu_count(), "numba_num_threads": int(numba.config.NUMBA_NUM_THREADS),
            "numba_threading_layer": _layer()}


def _layer() -> str:
    try:
        import numba

        return str(numba.threading_layer())
    except Exception:  # only known after the first parallel call
        return "unset"
