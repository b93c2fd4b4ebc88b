"""Shared pytest setup.

Markers: ``gpu`` tests need a B200 (they run through the CUDA C-ABI library);
everything else runs on the CPU build container.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle

    oracle.lib()
    return oracle


def fill_case(golden, idx):
    """Unpack fill fixture ``idx`` (see tests/golden/make_golden.py: add_fill)."""
    pre = f"fill_{idx}_"
    s = golden[pre + "scalars"]
    return dict(
        name=str(golden["fill_names"][idx]),
        x0=golden[pre + "x0"],
        v_prev=float(s[0]), r=float(s[1]), eps=float(s[2]),
        lower=float(s[3]), upper=float(s[4]), anchor=float(s[5]),
        j_star=int(s[6]), m_grid=int(s[7]), n_sim=int(s[8]), prefix=bool(s[9]),
        ranges=[tuple(map(float, rr)) for rr in golden[pre + "ranges"]],
        seed=int(golden[pre + "seed"][0]),
        S_all=golden[pre + "S_all"], steps_all=golden[pre + "steps_all"],
        ss_ok=golden[pre + "ss_ok"], P=golden[pre + "P"], stats=golden[pre + "stats"],
        result=golden[pre + "result"],
    )


def bis_case(golden, idx):
    pre = f"bis_{idx}_"
    s = golden[pre + "scalars"]
    return dict(
        name=str(golden["bis_names"][idx]),
        x0=golden[pre + "x0"],
        v_prev=float(s[0]), r=float(s[1]), eps=float(s[2]),
        lower=float(s[3]), upper=float(s[4]), anchor=float(s[5]),
        j_star=int(s[6]), n_kappa=int(s[7]), n_sim=int(s[8]),
        ranges=[tuple(map(float, rr)) for rr in golden[pre + "ranges"]],
        seed=int(golden[pre + "seed"][0]),
        result=golden[pre + "result"], per=golden[pre + "per"], paths=golden[pre + "paths"],
    )


def lin_case(golden, idx):
    pre = f"lin_{idx}_"
    s = golden[pre + "scalars"]
    A = golden[pre + "A"]
    n = A.shape[0]
    bcd = golden[pre + "BCD"]
    return dict(name=str(golden["lin_names"][idx]), A=A, B=bcd[:n], C=bcd[n:2 * n],
                D=float(bcd[2 * n]), gain=float(bcd[2 * n + 1]), x0=golden[pre + "x0"],
                v_prev=float(s[0]), r=float(s[1]), eps=float(s[2]), lower=float(s[3]),
                upper=float(s[4]), anchor=float(s[5]), j_star=int(s[6]), m_grid=int(s[7]),
                n_sim=int(s[8]), mag=float(s[9]), seed=int(golden[pre + "seed"][0]),
                S_all=golden[pre + "S_all"], steps_all=golden[pre + "steps_all"],
                P=golden[pre + "P"], stats=golden[pre + "stats"],
                results=golden[pre + "results"])


def n_fill_cases(golden):
    return len(golden["fill_names"])


def n_bis_cases(golden):
    return len(golden["bis_names"])
