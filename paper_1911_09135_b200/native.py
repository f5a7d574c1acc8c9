"""ctypes binding of libsimtgraph_cuda.so (include/simtgraph_cuda.h).

The library is built in-tree (``paper_1911_09135_b200/_lib``) by
``python -m paper_1911_09135_b200.build`` / ``__graft_entry__.build()``.
There is no fallback: if the library or a CUDA device is missing, every
entry point raises ``SimtGraphError`` (loud failure, never a CPU path).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import ConfigError, ConvergenceError, ParseError, RangeError, SimtGraphError

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libsimtgraph_cuda.so"

SG_OK, SG_ECONFIG, SG_ERANGE, SG_ECONVERGE, SG_ECUDA, SG_ENOMEM = 0, -1, -2, -3, -4, -5
SG_EPARSE, SG_EIO = -6, -7
FLAG_TIMING, FLAG_PROFILE, FLAG_TWC_CLASSIC, FLAG_RELABEL, FLAG_NO_RELABEL = 1, 2, 4, 8, 16
APP_IDS = {"bfs": 0, "sssp": 1, "cc": 2, "pr": 3, "kcore": 4}
SCHED_IDS = {"alb": 0, "twc": 1, "lb": 2, "vertex": 3, "edge": 4}

EXPORTS = (
    "sg_last_error", "sg_device_count", "sg_graph_create", "sg_graph_create_rmat",
    "sg_graph_attach_random_weights", "sg_graph_with_weights", "sg_graph_info",
    "sg_graph_download", "sg_graph_view_size", "sg_graph_destroy", "sg_run", "sg_run_profiled",
    "sg_lb_kernel", "sg_nccl_unique_id", "sg_dist_run", "sg_dist_run_threads",
    "sg_twc_kernel", "sg_vertex_kernel", "sg_edge_kernel", "sg_kernel_launches",
    "sg_host_alloc", "sg_host_free", "sg_release_cached", "sg_run_cta_counts",
    "sg_graph_load_sgb1", "sg_nccl_release", "sg_graph_release_views", "sg_graph_build_ms",
    "sg_graph_partition", "sg_graph_part_info", "sg_team_create", "sg_team_connect",
    "sg_team_run", "sg_team_destroy", "sg_peer_run_threads", "sg_set_device",
)


class Params(ctypes.Structure):
    _fields_ = [("app", ctypes.c_int32), ("sched", ctypes.c_int32), ("blocked", ctypes.c_int32),
                ("devices", ctypes.c_int32), ("source", ctypes.c_int64), ("k", ctypes.c_int64),
                ("damping", ctypes.c_double), ("tol", ctypes.c_double),
                ("threshold", ctypes.c_int64), ("max_rounds", ctypes.c_int64),
                ("flags", ctypes.c_int32), ("reserved", ctypes.c_int32)]


ROUND_DTYPE = np.dtype([("frontier_size", "<i8"), ("active_edges", "<i8"), ("huge_count", "<i8"),
                        ("huge_edges", "<i8"), ("large_count", "<i8"), ("large_edges", "<i8"),
                        ("updated", "<i8"), ("comm_sent", "<i8"), ("comm_broadcast", "<i8"),
                        ("launches_twc", "<i8"), ("launches_lb", "<i8")])


class KernelTime(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_int64), ("ms", ctypes.c_double)]

_lib = None
_lock = threading.Lock()


def load(path: Path | None = None):
    """Load the library (once).  Raises SimtGraphError if it is not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path or os.environ.get("SIMTGRAPH_CUDA_LIB", LIB_PATH))
        if not p.exists():
            raise SimtGraphError(
                f"{p} not built: run `python -m paper_1911_09135_b200.build` (no CPU fallback)")
        lib = ctypes.CDLL(str(p))
        P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        pp = ctypes.POINTER(ctypes.c_void_p)
        sig = {
            "sg_last_error": ([], ctypes.c_char_p),
            "sg_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
            "sg_graph_create": ([P, P, P, i64, i64, pp], ctypes.c_int),
            "sg_graph_create_rmat": ([i32, i64, P, P, pp], ctypes.c_int),
            "sg_graph_attach_random_weights": ([P, P, i64, i64, pp], ctypes.c_int),
            "sg_graph_with_weights": ([P, P, pp], ctypes.c_int),
            "sg_graph_info": ([P, P, P, P], ctypes.c_int),
            "sg_graph_download": ([P, i32, P, P, P], ctypes.c_int),
            "sg_graph_view_size": ([P, i32, P], ctypes.c_int),
            "sg_graph_destroy": ([P], None),
            "sg_run": ([P, ctypes.POINTER(Params), P, P, i64, P, P], ctypes.c_int),
            "sg_run_profiled": ([P, ctypes.POINTER(Params), P, P, i64, P, P, P, i32, P],
                                ctypes.c_int),
            "sg_lb_kernel": ([P, i64, P, i64, P, i64, P, P, i64, P, P, P, i64, i32, i32, i32, i32,
                              i32, P, P, P], ctypes.c_int),
            "sg_twc_kernel": ([P, i64, P, i64, P, i64, P, i64, P, i64, P, i64, P, P, P, i64, i32,
                               i32, i32, i32, P], ctypes.c_int),
            "sg_vertex_kernel": ([P, i64, P, i64, P, i64, P, i64, P, P, P, i64, i32, i32, i32, P],
                                 ctypes.c_int),
            "sg_edge_kernel": ([P, i64, P, i64, P, i64, P, i64, P, P, P, i64, i32, i32, i32, P],
                               ctypes.c_int),
            "sg_kernel_launches": ([], ctypes.c_int64),
            "sg_nccl_unique_id": ([P], ctypes.c_int),
            "sg_dist_run": ([P, ctypes.POINTER(Params), P, i32, i32, P, P, i64, P, P],
                            ctypes.c_int),
            "sg_dist_run_threads": ([P, ctypes.POINTER(Params), i32, P, P, i64, P, P],
                                    ctypes.c_int),
            "sg_run_cta_counts": ([P, ctypes.POINTER(Params), P, P, i64, P, P, P, i64, P],
                                  ctypes.c_int),
            "sg_host_alloc": ([i64, pp], ctypes.c_int),
            "sg_host_free": ([P], None),
            "sg_release_cached": ([], None),
            "sg_graph_load_sgb1": ([ctypes.c_char_p, pp], ctypes.c_int),
            "sg_nccl_release": ([], None),
            "sg_graph_release_views": ([P], ctypes.c_int),
            "sg_graph_build_ms": ([P, P], ctypes.c_int),
            "sg_set_device": ([i32], ctypes.c_int),
            "sg_graph_partition": ([P, i32, i32, i32, pp], ctypes.c_int),
            "sg_graph_part_info": ([P, P, P, P, P, P], ctypes.c_int),
            "sg_team_create": ([i32, i32, i64, pp, P], ctypes.c_int),
            "sg_team_connect": ([P, P], ctypes.c_int),
            "sg_team_run": ([P, P, ctypes.POINTER(Params), P, P, i64, P, P], ctypes.c_int),
            "sg_team_destroy": ([P], None),
            "sg_peer_run_threads": ([P, ctypes.POINTER(Params), i32, P, P, i64, P, P],
                                    ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


class _PinnedBlock:
    """A cached pinned host block (sg_host_alloc); returned to the library's
    pool when the last numpy view of it is gone."""

    __slots__ = ("ptr", "__weakref__")

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        check(load().sg_host_alloc(nbytes, ctypes.byref(p)))
        self.ptr = p.value

    def __del__(self):
        if self.ptr and _lib is not None:
            _lib.sg_host_free(self.ptr)
            self.ptr = None


PINNED_MIN_BYTES = 4 << 20  # below this a pageable copy costs less than pinning


def pinned_empty(n: int, dtype) -> np.ndarray:
    """numpy array in pinned host memory (device->host copies at full PCIe speed)."""
    dtype = np.dtype(dtype)
    nbytes = max(int(n) * dtype.itemsize, 1)
    if nbytes < PINNED_MIN_BYTES:
        return np.empty(int(n), dtype=dtype)
    blk = _PinnedBlock(nbytes)
    raw = (ctypes.c_char * nbytes).from_address(blk.ptr)
    raw.owner = blk  # the array keeps the block alive
    return np.frombuffer(raw, dtype=dtype, count=int(n))


def release_cached():
    """Return the library's cached device blocks to the CUDA driver."""
    load().sg_release_cached()


def check(code: int):
    if code == SG_OK:
        return
    msg = (load().sg_last_error() or b"").decode(errors="replace")
    if code == SG_ECONFIG:
        raise ConfigError(msg)
    if code == SG_ERANGE:
        raise RangeError(msg)
    if code == SG_ECONVERGE:
        raise ConvergenceError(msg)
    if code == SG_EPARSE:
        raise ParseError(msg)
    if code == SG_EIO:
        raise OSError(msg)
    raise SimtGraphError(f"CUDA backend error {code}: {msg}")


def ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def device_count() -> int:
    n = ctypes.c_int(0)
    check(load().sg_device_count(ctypes.byref(n)))
    return n.value


def set_device(device: int):
    """Select the CUDA device for this thread's later library calls."""
    check(load().sg_set_device(int(device)))


def kernel_launches() -> int:
    return int(load().sg_kernel_launches())


class DeviceGraph:
    """Owning handle of an HBM-resident graph (sg_graph*)."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle

    @property
    def handle(self):
        if not self._h:
            raise SimtGraphError("device graph already released")
        return self._h

    def __del__(self):
        try:
            if self._h and _lib is not None:
                _lib.sg_graph_destroy(self._h)
        except Exception:  # pragma: no cover - interpreter teardown
            pass
        self._h = None

    def info(self):
        nv, ne, w = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        check(load().sg_graph_info(self.handle, ctypes.byref(nv), ctypes.byref(ne),
                                   ctypes.byref(w)))
        return nv.value, ne.value, bool(w.value)

    @classmethod
    def from_csr(cls, offsets, targets, weights=None):
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        targets = np.ascontiguousarray(targets, dtype=np.int32)
        if weights is not None:
            weights = np.ascontiguousarray(weights, dtype=np.int64)
        h = ctypes.c_void_p()
        check(load().sg_graph_create(ptr(offsets), ptr(targets), ptr(weights), len(offsets) - 1,
                                     len(targets), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def load_sgb1(cls, path):
        """SGB1 file straight into HBM (sg_graph_load_sgb1)."""
        h = ctypes.c_void_p()
        check(load().sg_graph_load_sgb1(os.fsencode(path), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def rmat(cls, scale, edge_factor, seed, probs):
        pcg = pcg64_words(seed)
        cuts = np.ascontiguousarray(np.cumsum(np.asarray(probs, dtype=np.float64))[:3])
        h = ctypes.c_void_p()
        check(load().sg_graph_create_rmat(scale, edge_factor, ptr(pcg), ptr(cuts), ctypes.byref(h)))
        return cls(h)

    def with_random_weights(self, seed, low, high):
        pcg = pcg64_words(seed)
        h = ctypes.c_void_p()
        check(load().sg_graph_attach_random_weights(self.handle, ptr(pcg), low, high,
                                                    ctypes.byref(h)))
        return DeviceGraph(h)

    def with_weights(self, weights):
        weights = np.ascontiguousarray(weights, dtype=np.int64)
        h = ctypes.c_void_p()
        check(load().sg_graph_with_weights(self.handle, ptr(weights), ctypes.byref(h)))
        return DeviceGraph(h)

    def release_views(self):
        """Drop the cached derived layouts (CSC, symmetrized, relabeled store,
        exact pr layouts); they are rebuilt on demand."""
        check(load().sg_graph_release_views(self.handle))

    def build_ms(self):
        """Last build times (ms) of {csc, sym, relabel, exact}."""
        out = np.zeros(4, dtype=np.float64)
        check(load().sg_graph_build_ms(self.handle, ptr(out)))
        return dict(zip(("csc", "sym", "relabel", "exact"), out.tolist()))

    def download(self, which=0, weights=False):
        """Host copies of a view: 0 CSR, 1 CSC, 2 symmetrized CSR."""
        nv, ne, _ = self.info()
        vne = ctypes.c_int64()
        check(load().sg_graph_view_size(self.handle, which, ctypes.byref(vne)))
        off = np.empty(nv + 1, dtype=np.int64)
        tgt = np.empty(vne.value, dtype=np.int32)
        w = np.empty(ne, dtype=np.int64) if weights else None
        check(load().sg_graph_download(self.handle, which, ptr(off), ptr(tgt), ptr(w)))
        return off, tgt, w

    def run(self, params: Params, rounds_cap=1 << 16, profile=False):
        """Run the BSP loop on the device.  Returns (labels, round log, ms) or,
        with ``profile``, (labels, round log, ms, {kernel: (launches, ms)}).
        A run longer than ``rounds_cap`` rounds is repeated with a log large
        enough for all of it (runs are deterministic), never truncated."""
        nv, _, _ = self.info()
        labels = pinned_empty(nv, np.float64)
        while True:
            rounds = np.zeros(max(int(rounds_cap), 1), dtype=ROUND_DTYPE)
            n = ctypes.c_int64(0)
            ms = ctypes.c_double(0.0)
            kt = (KernelTime * 64)()
            nkt = ctypes.c_int32(0)
            if profile:
                code = load().sg_run_profiled(self.handle, ctypes.byref(params), ptr(labels),
                                              ptr(rounds), len(rounds), ctypes.byref(n),
                                              ctypes.byref(ms), kt, 64, ctypes.byref(nkt))
            else:
                code = load().sg_run(self.handle, ctypes.byref(params), ptr(labels), ptr(rounds),
                                     len(rounds), ctypes.byref(n), ctypes.byref(ms))
            if n.value <= len(rounds) or code not in (SG_OK, SG_ECONVERGE):
                break
            rounds_cap = n.value
        log = rounds[: min(n.value, len(rounds))].copy()
        if code == SG_ECONVERGE:
            err = ConvergenceError((load().sg_last_error() or b"").decode())
            err.metrics_log = log
            raise err
        check(code)
        if profile:
            kernels = {kt[i].name.decode(): (int(kt[i].launches), float(kt[i].ms))
                       for i in range(nkt.value)}
            return labels, log, ms.value, kernels
        return labels, log, ms.value

    def run_cta_counts(self, params: Params, rounds_cap=1 << 16, cta_rounds=512):
        """sg_run with hardware load counters: (labels, log, ms, cta) where
        cta[r, c] = edges processed by CTA slot c in round r (first cta_rounds)."""
        nv, _, _ = self.info()
        labels = pinned_empty(nv, np.float64)
        rounds = np.zeros(rounds_cap, dtype=ROUND_DTYPE)
        n = ctypes.c_int64(0)
        ms = ctypes.c_double(0.0)
        g = ctypes.c_int32(0)
        cta = np.zeros(cta_rounds * 4096, dtype=np.uint64)  # room for <= 512 SMs x 8 CTAs
        check(load().sg_run_cta_counts(self.handle, ctypes.byref(params), ptr(labels),
                                       ptr(rounds), rounds_cap, ctypes.byref(n),
                                       ctypes.byref(ms), ptr(cta), cta_rounds, ctypes.byref(g)))
        log = rounds[: min(n.value, rounds_cap)].copy()
        r = min(len(log), cta_rounds)
        return labels, log, ms.value, cta[: r * g.value].reshape(r, g.value).astype(np.int64)


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    check(load().sg_nccl_unique_id(buf))
    return bytes(buf)


def nccl_release():
    """Destroy the NCCL communicators sg_dist_run cached (one per id / rank /
    world / device); call before tearing down the process group."""
    load().sg_nccl_release()


def dist_run(dev: DeviceGraph, params: Params, nccl_id: bytes, rank: int, world: int,
             rounds_cap=1 << 16):
    """One edge-cut partition per rank over NCCL (sg_dist_run); every rank gets
    the merged labels and the global round log."""
    nv, _, _ = dev.info()
    labels = pinned_empty(nv, np.float64)
    rounds = np.zeros(rounds_cap, dtype=ROUND_DTYPE)
    n = ctypes.c_int64(0)
    ms = ctypes.c_double(0.0)
    idb = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
    check(load().sg_dist_run(dev.handle, ctypes.byref(params), idb, rank, world, ptr(labels),
                             ptr(rounds), rounds_cap, ctypes.byref(n), ctypes.byref(ms)))
    return labels, rounds[: min(n.value, rounds_cap)].copy(), ms.value


def dist_run_threads(dev: DeviceGraph, params: Params, world: int, rounds_cap=1 << 16):
    """The per-rank edge-cut code path of sg_dist_run with `world` ranks as host
    threads on this one GPU (collectives are device kernels): rank 0's labels
    and the global round log."""
    nv, _, _ = dev.info()
    labels = pinned_empty(nv, np.float64)
    rounds = np.zeros(rounds_cap, dtype=ROUND_DTYPE)
    n = ctypes.c_int64(0)
    ms = ctypes.c_double(0.0)
    check(load().sg_dist_run_threads(dev.handle, ctypes.byref(params), world, ptr(labels),
                                     ptr(rounds), rounds_cap, ctypes.byref(n), ctypes.byref(ms)))
    return labels, rounds[: min(n.value, rounds_cap)].copy(), ms.value


def _run_with_log(call, nv, rounds_cap):
    """call(labels, rounds, n, ms) -> code; repeated with a larger round log
    when the run outgrew it (runs are deterministic), never truncated."""
    labels = pinned_empty(nv, np.float64)
    while True:
        rounds = np.zeros(max(int(rounds_cap), 1), dtype=ROUND_DTYPE)
        n = ctypes.c_int64(0)
        ms = ctypes.c_double(0.0)
        code = call(labels, rounds, n, ms)
        if n.value <= len(rounds) or code not in (SG_OK, SG_ECONVERGE):
            break
        rounds_cap = n.value
    log = rounds[: min(n.value, len(rounds))].copy()
    if code == SG_ECONVERGE:
        err = ConvergenceError((load().sg_last_error() or b"").decode())
        err.metrics_log = log
        raise err
    check(code)
    return labels, log, ms.value


PART_CSR, PART_CSC, PART_SYM = 0, 1, 2
PART_RELABEL, PART_NO_RELABEL = 0x100, 0x200  # block-local hot relabeling on / off
FLAG_RELABEL, FLAG_NO_RELABEL = 8, 16          # sg_params.flags


class DevicePartition(DeviceGraph):
    """One rank's edge-cut rows of a traversal view (sg_graph_partition):
    only rows [cuts[rank], cuts[rank+1]) and their edges live in HBM."""

    @classmethod
    def of(cls, dev: DeviceGraph, kind: int, world: int, rank: int):
        h = ctypes.c_void_p()
        check(load().sg_graph_partition(dev.handle, kind, world, rank, ctypes.byref(h)))
        return cls(h)

    def part_info(self):
        kind, rank, world = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        cuts = np.zeros(64, dtype=np.int64)
        full = ctypes.c_int64()
        check(load().sg_graph_part_info(self.handle, ctypes.byref(kind), ctypes.byref(rank),
                                        ctypes.byref(world), ptr(cuts), ctypes.byref(full)))
        return {"kind": kind.value, "rank": rank.value, "world": world.value,
                "cuts": cuts[: world.value + 1].copy(), "full_edges": full.value}


class Team:
    """One rank's symmetric HBM region of the NVLink peer transport
    (sg_team_create / sg_team_connect): every rank exports its region as a
    CUDA IPC handle, the handles are exchanged out of band, and each rank maps
    its peers' regions.  Runs are sg_team_run on this rank's partition."""

    def __init__(self, rank: int, world: int, num_vertices: int, host_sync=None):
        # host_sync: a collective the ranks run before each sg_team_run (e.g. the
        # process group's barrier), so no rank's device barrier starts spinning
        # while a peer is still busy on the host (the device barrier gives up
        # after 60 s and the team is then unusable)
        self.host_sync = host_sync
        self._h = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 64)()
        check(load().sg_team_create(rank, world, num_vertices, ctypes.byref(self._h), buf))
        self.handle_bytes = bytes(buf)
        self.rank, self.world, self.num_vertices = rank, world, num_vertices

    def connect(self, handles):
        blob = b"".join(bytes(h) for h in handles)
        if len(blob) != 64 * self.world:
            raise SimtGraphError("need one 64-byte IPC handle per rank")
        arr = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        check(load().sg_team_connect(self._h, arr))

    def run(self, part: DevicePartition, params: Params, rounds_cap=1 << 16):
        nv, _, _ = part.info()
        if self.host_sync is not None:
            self.host_sync()
        return _run_with_log(
            lambda lab, rounds, n, ms: load().sg_team_run(
                self._h, part.handle, ctypes.byref(params), ptr(lab), ptr(rounds), len(rounds),
                ctypes.byref(n), ctypes.byref(ms)), nv, rounds_cap)

    def close(self):
        if self._h and _lib is not None:
            _lib.sg_team_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter teardown
            pass


def peer_run_threads(dev: DeviceGraph, params: Params, world: int, rounds_cap=1 << 16):
    """The NVLink peer transport with `world` ranks as host threads on this GPU
    (peers = the other ranks' regions in the same HBM): rank 0's labels and the
    global round log."""
    nv, _, _ = dev.info()
    return _run_with_log(
        lambda lab, rounds, n, ms: load().sg_peer_run_threads(
            dev.handle, ctypes.byref(params), world, ptr(lab), ptr(rounds), len(rounds),
            ctypes.byref(n), ctypes.byref(ms)), nv, rounds_cap)


def pcg64_words(seed) -> np.ndarray:
    """(state_hi, state_lo, inc_hi, inc_lo) of np.random.PCG64(seed)."""
    st = np.random.PCG64(seed).state["state"]
    m = (1 << 64) - 1
    s, inc = st["state"], st["inc"]
    return np.array([s >> 64, s & m, inc >> 64, inc & m], dtype=np.uint64)
