"""Kernel-level plugin: the reference backend protocol on the B200.

Same module protocol as the reference's ``_kernels_py`` / ``_kernels``
(selected by kernels.get_backend, kernels.py:16-41): ``BACKEND_NAME``,
``OP_*``, ``probe_depths`` and the four kernels with the reference's
positional signatures (_kernels_py.py:88-201).  Buffers are the caller's
numpy arrays; ``out``, ``per_cta_edges`` and ``per_warp_paths`` are mutated
in place, ``lb_kernel`` returns the modeled search-access count.  Each call
copies its inputs to HBM, runs the sg_*_kernel CUDA kernels and copies the
mutated buffers back, so the reference's own engine can drive the B200
kernels round by round (the parity harness of SURVEY §8b).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import native

BACKEND_NAME = "cuda"
OP_BFS = 0
OP_SSSP = 1
OP_CC = 2
OP_PULL_ADD = 3

_depths: dict[int, np.ndarray] = {}


def probe_depths(n: int) -> np.ndarray:
    """Bisection probe count per landing segment of an n-entry prefix (_kernels_py.py:34-56)."""
    d = _depths.get(n)
    if d is None:
        d = np.zeros(n, dtype=np.int64)
        todo = [(0, n - 1, 0)]
        while todo:
            lo, hi, k = todo.pop()
            if lo == hi:
                d[lo] = k
            else:
                mid = (lo + hi) // 2
                todo += [(lo, mid, k + 1), (mid + 1, hi, k + 1)]
        _depths[n] = d
    return d


def _c(a, dtype):
    a = np.asarray(a)
    if a.dtype != dtype or not a.flags.c_contiguous:
        a = np.ascontiguousarray(a, dtype=dtype)
    return a


def _inout(a, dtype, name):
    if not isinstance(a, np.ndarray) or a.dtype != dtype or not a.flags.c_contiguous:
        raise TypeError(f"{name} must be a contiguous {np.dtype(dtype)} numpy array (mutated in place)")
    return a


def _graph(offsets, targets, weights):
    off = _c(offsets, np.int64)
    tgt = _c(targets, np.int32)
    w = _c(weights, np.float64) if weights is not None else np.empty(0, np.float64)
    return off, tgt, w


def lb_kernel(offsets, targets, weights, huge, cumulative, values, out, aux, opcode, blocked,
              num_ctas, threads_per_cta, warp_size, per_cta_edges, per_warp_paths):
    off, tgt, w = _graph(offsets, targets, weights)
    huge = _c(huge, np.int64)
    cum = _c(cumulative, np.int64)
    values = _c(values, np.float64)
    aux = _c(aux, np.float64)
    out = _inout(out, np.float64, "out")
    pce = _inout(per_cta_edges, np.int64, "per_cta_edges")
    pwp = _inout(per_warp_paths, np.int64, "per_warp_paths")
    acc = ctypes.c_int64(0)
    native.check(native.load().sg_lb_kernel(
        native.ptr(off), len(off) - 1, native.ptr(tgt), len(tgt), native.ptr(w), len(w),
        native.ptr(huge), native.ptr(cum), len(cum), native.ptr(values), native.ptr(out),
        native.ptr(aux), len(aux), int(opcode), int(blocked), int(num_ctas),
        int(threads_per_cta), int(warp_size), native.ptr(pce), native.ptr(pwp),
        ctypes.byref(acc)))
    return acc.value


def twc_kernel(offsets, targets, weights, small, medium, large, values, out, aux, opcode,
               num_ctas, threads_per_cta, warp_size, per_cta_edges):
    off, tgt, w = _graph(offsets, targets, weights)
    small, medium, large = (_c(x, np.int64) for x in (small, medium, large))
    values = _c(values, np.float64)
    aux = _c(aux, np.float64)
    out = _inout(out, np.float64, "out")
    pce = _inout(per_cta_edges, np.int64, "per_cta_edges")
    native.check(native.load().sg_twc_kernel(
        native.ptr(off), len(off) - 1, native.ptr(tgt), len(tgt), native.ptr(w), len(w),
        native.ptr(small), len(small), native.ptr(medium), len(medium), native.ptr(large),
        len(large), native.ptr(values), native.ptr(out), native.ptr(aux), len(aux), int(opcode),
        int(num_ctas), int(threads_per_cta), int(warp_size), native.ptr(pce)))


def vertex_kernel(offsets, targets, weights, frontier, values, out, aux, opcode, num_ctas,
                  threads_per_cta, per_cta_edges):
    off, tgt, w = _graph(offsets, targets, weights)
    fr = _c(frontier, np.int64)
    values = _c(values, np.float64)
    aux = _c(aux, np.float64)
    out = _inout(out, np.float64, "out")
    pce = _inout(per_cta_edges, np.int64, "per_cta_edges")
    native.check(native.load().sg_vertex_kernel(
        native.ptr(off), len(off) - 1, native.ptr(tgt), len(tgt), native.ptr(w), len(w),
        native.ptr(fr), len(fr), native.ptr(values), native.ptr(out), native.ptr(aux), len(aux),
        int(opcode), int(num_ctas), int(threads_per_cta), native.ptr(pce)))


def edge_kernel(offsets, targets, weights, frontier, values, out, aux, opcode, num_ctas,
                threads_per_cta, per_cta_edges):
    off, tgt, w = _graph(offsets, targets, weights)
    fr = _c(frontier, np.int64)
    values = _c(values, np.float64)
    aux = _c(aux, np.float64)
    out = _inout(out, np.float64, "out")
    pce = _inout(per_cta_edges, np.int64, "per_cta_edges")
    native.check(native.load().sg_edge_kernel(
        native.ptr(off), len(off) - 1, native.ptr(tgt), len(tgt), native.ptr(w), len(w),
        native.ptr(fr), len(fr), native.ptr(values), native.ptr(out), native.ptr(aux), len(aux),
        int(opcode), int(num_ctas), int(threads_per_cta), native.ptr(pce)))
