"""Multi-GPU edge cut: one process per GPU (torchrun), NCCL over NVLink.

The reference simulates devices in one process (engine.py:64-113, 215-234);
here each rank owns one contiguous edge-balanced row block of the traversal
view (the same cuts as ``engine.edge_cut_bounds``), runs the ALB round on its
local frontier, and ``sg_dist_run`` exchanges labels with ncclAllReduce(min)
plus a device-side diff and an all-reduced quiescence counter.  torch is only
plumbing here: the process group shares the 128-byte NCCL id and reduces the
per-rank step times (max over ranks).
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


def partition_bounds(offsets: np.ndarray, world: int):
    """Row blocks [start, end) per rank — identical to the reference's make_partition."""
    from .engine import edge_cut_bounds
    return edge_cut_bounds(offsets, world)
