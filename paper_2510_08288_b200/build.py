"""Build the sm_100a library in-tree: ``python -m paper_2510_08288_b200.build``.

nvcc cross-compiles without a GPU; the .so lands in ``_lib/`` next to this
file (git-ignored, shipped to the GPU box with the working tree).
"""

from __future__ import annotations

import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIB = HERE / "_lib" / "librefgov_b200.so"


def build(force: bool = False) -> Path:
    cmd = ["make", "-s", "-j8", "-C", str(CSRC)]
    if force:
        cmd.append("-B")
    subprocess.run(cmd, check=True)
    if not LIB.exists():
        raise RuntimeError(f"build did not produce {LIB}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
