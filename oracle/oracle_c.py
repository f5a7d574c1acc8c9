"""ctypes wrapper for the C oracle (``sg_oracle.c``) — TEST INFRASTRUCTURE ONLY.

Used by tests/ (mid-size parity where the numpy oracle is slow), by
``__graft_entry__.smoke()`` as the checker, and by ``bench.py`` for the
``cpu_baseline`` / ``--impl reference`` legs.  Cross-validated against the
numpy oracle (itself pinned to tests/golden) in tests/test_oracle.py.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libsgoracle.so"
APP_IDS = {"bfs": 0, "sssp": 1, "cc": 2, "pr": 3, "kcore": 4}

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        _lib.sgo_run.argtypes = [ctypes.c_int, i64, P, P, P, P, P, i64, i64, ctypes.c_double,
                                 ctypes.c_double, i64, ctypes.c_int, P, P, i64,
                                 ctypes.POINTER(i64)]
        _lib.sgo_run.restype = ctypes.c_int
        _lib.sgo_rmat_pairs.argtypes = [ctypes.c_int, i64, ctypes.c_uint64, ctypes.c_uint64,
                                        ctypes.c_uint64, ctypes.c_uint64, P, P, P, ctypes.c_int]
        _lib.sgo_rmat_pairs.restype = None
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def run(app, view_off, view_tgt, view_w=None, graph_off=None, graph_tgt=None, *, source=0,
        k=2, damping=0.85, tol=1e-6, max_rounds=0, threads=1):
    """Run one app.  The caller supplies the traversal view exactly as
    engine.run builds it (CSR / sym CSR for push, CSC for pr, sym CSR for
    kcore) and the app graph CSR for pr (out-degrees) / kcore (neighbours).
    Returns (labels float64, log int64[rounds, 2], status)."""
    nv = len(view_off) - 1
    labels = np.empty(nv, dtype=np.float64)
    cap = 1 << 16
    log = np.zeros((cap, 2), dtype=np.int64)
    n = ctypes.c_int64(0)
    view_off = np.ascontiguousarray(view_off, dtype=np.int64)
    view_tgt = np.ascontiguousarray(view_tgt, dtype=np.int32)
    if view_w is not None:
        view_w = np.ascontiguousarray(view_w, dtype=np.float64)
    if graph_off is None:
        graph_off, graph_tgt = view_off, view_tgt
    graph_off = np.ascontiguousarray(graph_off, dtype=np.int64)
    graph_tgt = np.ascontiguousarray(graph_tgt, dtype=np.int32)
    st = lib().sgo_run(APP_IDS[app], nv, _p(view_off), _p(view_tgt), _p(view_w), _p(graph_off),
                       _p(graph_tgt), source, k, damping, tol, max_rounds, threads, _p(labels),
                       _p(log), cap, ctypes.byref(n))
    return labels, log[: min(n.value, cap)].copy(), st


def rmat_pairs(scale, edge_factor=16, seed=1, probs=(0.57, 0.19, 0.19, 0.05), threads=0):
    """Same edge stream as numpy's generate_rmat (graph.py:274-298), multi-threaded."""
    st = np.random.PCG64(seed).state["state"]
    s, inc = st["state"], st["inc"]
    ne = edge_factor << scale
    cuts = np.ascontiguousarray(np.cumsum(np.asarray(probs, dtype=np.float64))[:3])
    src = np.empty(ne, dtype=np.int32)
    dst = np.empty(ne, dtype=np.int32)
    m = (1 << 64) - 1
    lib().sgo_rmat_pairs(scale, ne, s >> 64, s & m, inc >> 64, inc & m, _p(cuts), _p(src),
                         _p(dst), threads or (os.cpu_count() or 1))
    return src, dst


def prepare(off, tgt, weights, app):
    """(view_off, view_tgt, view_w, graph_off, graph_tgt) as engine.run would use."""
    from . import oracle_np as O
    if app in ("cc", "kcore"):
        off, tgt, weights = O.symmetrize(off, tgt, weights)
    if app == "pr":
        voff, vtgt, _ = O.transpose(off, tgt)
        return voff, vtgt, None, off, tgt
    w = None
    if app == "sssp" and weights is not None:
        w = weights.astype(np.float64)
    return off, tgt, w, off, tgt


def csr_from_pairs(src, dst, nv, weights=None):
    """Stable counting-sort CSR (== graph.py:63-76 from_edges)."""
    L = lib()
    if not hasattr(L, "_csr_sig"):
        P = ctypes.c_void_p
        L.sgo_csr_from_pairs.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P, P, P, P]
        L.sgo_csr_from_pairs.restype = None
        L._csr_sig = True
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    off = np.empty(nv + 1, dtype=np.int64)
    tgt = np.empty(len(src), dtype=np.int32)
    w_out = None
    if weights is not None:
        weights = np.ascontiguousarray(weights, dtype=np.int64)
        w_out = np.empty(len(src), dtype=np.int64)
    L.sgo_csr_from_pairs(len(src), nv, _p(src), _p(dst), _p(weights), _p(off), _p(tgt), _p(w_out))
    return off, tgt, w_out


def _sig(name, args):
    L = lib()
    fn = getattr(L, name)
    if not getattr(fn, "_sg_sig", False):
        fn.argtypes = args
        fn.restype = None
        fn._sg_sig = True
    return fn


def transpose(off, tgt):
    """Stable CSC of a CSR (== Graph.csc(), graph.py:95-113), in C."""
    P = ctypes.c_void_p
    nv = len(off) - 1
    toff = np.empty(nv + 1, dtype=np.int64)
    ttgt = np.empty(len(tgt), dtype=np.int32)
    _sig("sgo_transpose", [ctypes.c_int64, P, P, P, P])(
        nv, _p(np.ascontiguousarray(off, dtype=np.int64)),
        _p(np.ascontiguousarray(tgt, dtype=np.int32)), _p(toff), _p(ttgt))
    return toff, ttgt


def symmetrize(off, tgt, coff=None, ctgt=None, threads=0):
    """Symmetrized CSR (== Graph.symmetrized(), graph.py:115-128), in C."""
    P = ctypes.c_void_p
    if coff is None:
        coff, ctgt = transpose(off, tgt)
    nv = len(off) - 1
    soff = np.empty(nv + 1, dtype=np.int64)
    stgt = np.empty(len(tgt) + len(ctgt), dtype=np.int32)
    _sig("sgo_symmetrize", [ctypes.c_int64, P, P, P, P, P, P, ctypes.c_int])(
        nv, _p(off), _p(tgt), _p(coff), _p(ctgt), _p(soff), _p(stgt),
        threads or (os.cpu_count() or 1))
    return soff, stgt


def rmat_csr(scale, edge_factor=16, seed=1, probs=(0.57, 0.19, 0.19, 0.05), threads=0):
    """generate_rmat's CSR (graph.py:274-298) built in C (multi-threaded stream)."""
    src, dst = rmat_pairs(scale, edge_factor, seed, probs, threads)
    off, tgt, _ = csr_from_pairs(src, dst, 1 << scale)
    return off, tgt
