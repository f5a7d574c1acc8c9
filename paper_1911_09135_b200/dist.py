"""Multi-GPU edge cut: one process per GPU (torchrun).

The reference simulates devices in one process (engine.py:64-113, 215-234);
here each rank owns one contiguous edge-balanced row block of the traversal
view (the same cuts as ``engine.edge_cut_bounds``) and runs the ALB round on
its local frontier.  Two transports:

* **peer** (default, ``run_app_peer``): the B200 path.  A rank stores only its
  own rows (``partition``), keeps its labels in a symmetric HBM region whose
  CUDA IPC handle the other ranks map (``make_team``), and the round's own
  kernels store label updates straight into the owners' / mirrors' memory over
  NVLink, with a device-side barrier and quiescence test: one CUDA-graph
  launch per run, no collective library inside the loop (sg_peer.cu).
* **nccl** (``run_app``): every rank holds the whole graph; labels are
  exchanged with NCCL (sparse alltoallv of updated mirrors or all-reduce(min))
  and rounds are driven from the host (sg_dist.cu / sg_dist_push.cu).

torch is only plumbing: the process group exchanges the 64-byte IPC handles
(or the NCCL id) and reduces the per-rank step times (max over ranks).
"""

from __future__ import annotations

import os

import numpy as np

from . import native
from .apps import make_app
from .engine import RunResult, device_params, records_from_log
from .errors import ConfigError
from .schedulers import Scheduler
from .simt import KernelConfig


def env():
    """(rank, local_rank, world) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def init_device() -> int:
    """Bind this process to its GPU (LOCAL_RANK modulo the visible devices),
    for the library's calls and torch's; returns the device index."""
    _, local, _ = env()
    dev = local % max(native.device_count(), 1)
    native.set_device(dev)
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.set_device(dev)
    except ImportError:  # pragma: no cover - torch is plumbing only
        pass
    return dev


def _tensor_device(dist):
    import torch
    return torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend() == "nccl" else torch.device("cpu")


def share_nccl_id(dist, make_id=None) -> bytes:
    """Rank 0 creates the NCCL unique id, every rank receives it (broadcast)."""
    import torch
    dev = _tensor_device(dist)
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if dist.get_rank() == 0:
        raw = (make_id or native.nccl_unique_id)()
        buf.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    dist.broadcast(buf, src=0)
    return bytes(buf.cpu().numpy().tobytes())


def max_over_ranks(dist, value: float) -> float:
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=_tensor_device(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def release():
    """Free the NCCL communicators the nccl transport cached (sg_nccl_release);
    call before destroy_process_group.  A communicator is reused by every run
    with the same id, so a caller that passes a fresh id per run should
    release after each."""
    native.nccl_release()


def run_app(graph, app_name: str, scheduler: Scheduler = Scheduler("alb"),
            config: KernelConfig = KernelConfig(), *, rank: int, world: int, nccl_id: bytes,
            max_rounds=None, **params) -> RunResult:
    """engine.run_app with one edge-cut partition per rank (every app)."""
    app = make_app(app_name, **params)
    if max_rounds is None:
        max_rounds = 10 * max(graph.num_vertices, 1) + 256
    p = device_params(app, scheduler, config, world, max_rounds)
    labels, log, ms = native.dist_run(graph.device(), p, nccl_id, rank, world)
    return RunResult(labels=labels, records=records_from_log(log, scheduler, config),
                     app_name=app.name, scheduler=scheduler, config=config, devices=world,
                     num_vertices=graph.num_vertices, num_edges=graph.num_edges,
                     device_ms=ms, round_log=log)


def run_app_threads(graph, app_name: str, scheduler: Scheduler = Scheduler("alb"),
                    config: KernelConfig = KernelConfig(), *, world: int, max_rounds=None,
                    **params) -> RunResult:
    """The same per-rank protocol with `world` ranks as threads on this GPU."""
    app = make_app(app_name, **params)
    if max_rounds is None:
        max_rounds = 10 * max(graph.num_vertices, 1) + 256
    p = device_params(app, scheduler, config, world, max_rounds)
    labels, log, ms = native.dist_run_threads(graph.device(), p, world)
    return RunResult(labels=labels, records=records_from_log(log, scheduler, config),
                     app_name=app.name, scheduler=scheduler, config=config, devices=world,
                     num_vertices=graph.num_vertices, num_edges=graph.num_edges,
                     device_ms=ms, round_log=log)


PART_KIND = {"bfs": native.PART_CSR, "sssp": native.PART_CSR, "pr": native.PART_CSC,
             "cc": native.PART_SYM, "kcore": native.PART_SYM}


class Partition:
    """This rank's rows of the traversal view an app runs on (Gluon's
    outgoing edge cut, the reference's make_partition cuts): only the block's
    edges (and weights) are stored in HBM, so the full graph may be dropped."""

    def __init__(self, graph, app_name: str, rank: int, world: int, relabel=None):
        if app_name not in PART_KIND:
            raise ConfigError(f"unknown app {app_name!r}")
        self.app_name = app_name
        self.num_vertices = graph.num_vertices
        self.num_edges = graph.num_edges
        self.rank, self.world = rank, world
        kind = PART_KIND[app_name] | (0 if relabel is None else
                                      native.PART_RELABEL if relabel else native.PART_NO_RELABEL)
        self._dev = native.DevicePartition.of(graph.device(), kind, world, rank)
        info = self._dev.part_info()
        self.kind, self.cuts, self.view_edges = info["kind"], info["cuts"], info["full_edges"]
        self.local_edges = self._dev.info()[1]

    def device(self):
        return self._dev

    @property
    def rows(self):
        return int(self.cuts[self.rank]), int(self.cuts[self.rank + 1])


def partition(graph, app_name: str, rank: int, world: int, relabel=None) -> Partition:
    """This rank's edge-cut rows for ``app_name`` (CSR for bfs / sssp, CSC for
    pr, symmetrized for cc / kcore).  ``relabel``: the block-local hot-vertex
    layout (True / False; None = automatic: skewed graphs of >= 2^20
    vertices); labels are returned in the original numbering either way."""
    return Partition(graph, app_name, rank, world, relabel)


def _all_gather_bytes(dist, data: bytes) -> list:
    import torch
    dev = _tensor_device(dist)
    t = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(dev)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [bytes(x.cpu().numpy().tobytes()) for x in out]


def make_team(dist, num_vertices: int) -> "native.Team":
    """This rank's symmetric region, connected to every peer's (the IPC
    handles travel through the torch process group)."""
    team = native.Team(dist.get_rank(), dist.get_world_size(), num_vertices,
                       host_sync=dist.barrier)
    team.connect(_all_gather_bytes(dist, team.handle_bytes))
    dist.barrier()
    return team


def run_app_peer(part: Partition, app_name: str, scheduler: Scheduler = Scheduler("alb"),
                 config: KernelConfig = KernelConfig(), *, team, max_rounds=None,
                 **params) -> RunResult:
    """engine.run_app for one rank of the NVLink peer transport: every rank
    calls it with its own partition and team; each returns the merged labels
    and the global round log (comm counters as the reference's devices=D run)."""
    if part.app_name != app_name:
        raise ConfigError(f"partition was cut for {part.app_name!r}, not {app_name!r}")
    app = make_app(app_name, **params)
    if max_rounds is None:
        max_rounds = 10 * max(part.num_vertices, 1) + 256
    p = device_params(app, scheduler, config, part.world, max_rounds)
    labels, log, ms = team.run(part.device(), p)
    return RunResult(labels=labels, records=records_from_log(log, scheduler, config),
                     app_name=app.name, scheduler=scheduler, config=config, devices=part.world,
                     num_vertices=part.num_vertices, num_edges=part.num_edges,
                     device_ms=ms, round_log=log)


def run_app_peer_threads(graph, app_name: str, scheduler: Scheduler = Scheduler("alb"),
                         config: KernelConfig = KernelConfig(), *, world: int, max_rounds=None,
                         relabel=None, **params) -> RunResult:
    """The peer transport with `world` ranks as threads on this GPU (each with
    its own partition and region): the multi-GPU kernels on one device."""
    app = make_app(app_name, **params)
    if max_rounds is None:
        max_rounds = 10 * max(graph.num_vertices, 1) + 256
    p = device_params(app, scheduler, config, world, max_rounds)
    if relabel is not None:
        p.flags |= native.FLAG_RELABEL if relabel else native.FLAG_NO_RELABEL
    labels, log, ms = native.peer_run_threads(graph.device(), p, world)
    return RunResult(labels=labels, records=records_from_log(log, scheduler, config),
                     app_name=app.name, scheduler=scheduler, config=config, devices=world,
                     num_vertices=graph.num_vertices, num_edges=graph.num_edges,
                     device_ms=ms, round_log=log)


def partition_bounds(offsets: np.ndarray, world: int):
    """Row blocks [start, end) per rank — identical to the reference's make_partition."""
    from .engine import edge_cut_bounds
    return edge_cut_bounds(offsets, world)
