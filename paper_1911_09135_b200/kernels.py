"""Kernel backend selection — the reference's plugin seam (kernels.py:16-41).

The only backend is ``cuda`` (``cuda_backend``: the four kernels of
_kernels_py.py:88-201 executed on the B200 through the C ABI).  There is no
numpy / Cython fallback; ``SIMTGRAPH_KERNELS`` may only name ``cuda``.
Importing this module does not touch the GPU; the library is loaded on the
first kernel call.
"""

from __future__ import annotations

import os

from . import cuda_backend
from .errors import ConfigError


def get_backend(name: str):
    if name == "cuda":
        return cuda_backend
    raise ConfigError(f"unknown kernel backend {name!r} (only 'cuda' exists)")


backend = get_backend(os.environ.get("SIMTGRAPH_KERNELS", "cuda"))
BACKEND_NAME = backend.BACKEND_NAME
OP_BFS = backend.OP_BFS
OP_SSSP = backend.OP_SSSP
OP_CC = backend.OP_CC
OP_PULL_ADD = backend.OP_PULL_ADD
