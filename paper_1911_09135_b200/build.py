"""Build libsimtgraph_cuda.so in-tree for sm_100a (``python -m paper_1911_09135_b200.build``).

nvcc cross-compiles without a GPU; the .so lands in ``_lib/`` and travels with
the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

CSRC = Path(__file__).resolve().parent / "csrc"


def build(verbose: bool = False) -> Path:
    jobs = str(min(8, os.cpu_count() or 1))
    cmd = ["make", "-C", str(CSRC), f"-j{jobs}"]
    if not verbose:
        cmd.append("-s")
    subprocess.run(cmd, check=True)
    lib = CSRC.parent / "_lib" / "libsimtgraph_cuda.so"
    if not lib.exists():
        raise RuntimeError(f"build did not produce {lib}")
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
