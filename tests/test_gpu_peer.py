"""GPU parity of the NVLink peer transport (sg_peer.cu): the multi-GPU edge cut
where each rank stores only its rows and the round's kernels write label
updates straight into the owners' / mirrors' HBM.  Driven on one B200 with
ranks as threads (peers = the other ranks' regions in the same HBM) and with
two torchrun processes (CUDA IPC mappings, the code path of one process per
GPU).  Bar: the reference's devices=D labels (sha256), per-round frontier /
edges, comm_sent / comm_broadcast and kernel launches (engine.py:205-235)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from test_gpu_parity import _check, _graph, _sched

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def sg():
    import paper_1911_09135_b200 as sg
    from paper_1911_09135_b200 import native
    if native.device_count() < 1:
        pytest.fail("no CUDA device visible")
    return sg


@pytest.mark.parametrize("gname,key", [("rmat12", "alb/d2"), ("rmat12", "alb/d4"),
                                       ("rmat12", "alb/d8"), ("rmat12", "alb-t256/d2"),
                                       ("rmat12", "alb-t256/d4"), ("rmat10", "lb/d2"),
                                       ("rmat10", "twc/d4"), ("rmat10", "alb-t64/d2"),
                                       ("uniform10", "alb/d3")])
@pytest.mark.parametrize("app", ["bfs", "sssp", "cc", "pr", "kcore"])
@pytest.mark.parametrize("relabel", [False, True])
def test_peer_ranks_as_threads(sg, golden, app, gname, key, relabel):
    """relabel: the block-local hot-vertex layout (each rank's block renumbered
    onto itself, rows sorted) -- same labels, logs and counters."""
    from paper_1911_09135_b200 import dist
    info = golden["runs"][gname][f"{app}/{key}"]
    g = _graph(sg, gname)
    if app == "sssp":
        g = sg.attach_random_weights(g, 2)
    world = int(key.split("/d")[1])
    res = dist.run_app_peer_threads(g, app, _sched(sg, "x/" + key.split("/")[0] + "/x"),
                                    world=world, relabel=relabel)
    _check(sg, res, info, app)
    if app == "pr":  # the exact-order pull: bit-identical to the reference
        assert [r.comm_broadcast for r in res.records] == [x[3] for x in info["per_round"]]


@pytest.mark.parametrize("app", ["bfs", "pr", "cc"])
def test_peer_partition_stores_only_its_rows(sg, app):
    """Each rank's partition holds exactly its block's edges; blocks are the
    reference's make_partition cuts (engine.py:64-75)."""
    from paper_1911_09135_b200 import dist
    from paper_1911_09135_b200.engine import edge_cut_bounds
    g = _graph(sg, "rmat12")
    view = {"bfs": 0, "pr": 1, "cc": 2}[app]
    off, _, _ = g.device().download(view)
    world = 4
    parts = [dist.partition(g, app, r, world) for r in range(world)]
    cuts = [a for a, _ in edge_cut_bounds(off, world)] + [g.num_vertices]
    assert [int(c) for c in parts[0].cuts] == cuts
    assert sum(p.local_edges for p in parts) == off[-1] == parts[0].view_edges
    for r, p in enumerate(parts):
        lo, hi = p.rows
        assert p.local_edges == off[hi] - off[lo]


def test_peer_partition_rejects_wrong_app(sg):
    from paper_1911_09135_b200 import dist, native
    from paper_1911_09135_b200.errors import ConfigError
    g = _graph(sg, "rmat10")
    part = dist.partition(g, "bfs", 0, 1)
    team = native.Team(0, 1, g.num_vertices)
    with pytest.raises(ConfigError):
        dist.run_app_peer(part, "pr", team=team)
    with pytest.raises(ConfigError):  # a partition is not a single-device graph
        native.DeviceGraph.run(part.device(), sg.engine.device_params(
            sg.apps.make_app("bfs"), sg.Scheduler("alb"), sg.KernelConfig(), 1, 100))


@pytest.mark.parametrize("gname,world", [("rmat12", 5), ("rmat12", 7), ("rmat14", 6),
                                         ("uniform10", 5)])
@pytest.mark.parametrize("app", ["bfs", "sssp", "cc", "pr", "kcore"])
@pytest.mark.parametrize("relabel", [False, True])
def test_peer_odd_worlds_match_d1(sg, golden, app, gname, world, relabel):
    """World sizes without goldens (cuts at arbitrary, unaligned ids; relabeled
    blocks with their edgeless / isolated tails): labels and the per-round
    frontier / active edges do not depend on D, so they must equal the
    reference's d1 run."""
    from paper_1911_09135_b200 import dist
    info = golden["runs"][gname][f"{app}/alb/d1"]
    g = _graph(sg, gname)
    if app == "sssp":
        g = sg.attach_random_weights(g, 2)
    res = dist.run_app_peer_threads(g, app, sg.Scheduler("alb"), world=world, relabel=relabel)
    assert sg.engine.labels_sha256(res.labels) == info["labels_sha256"]
    assert [[r.frontier_size, r.active_edges()] for r in res.records] == \
        [x[:2] for x in info["per_round"]]


@pytest.mark.parametrize("app", ["bfs", "sssp", "cc", "pr", "kcore"])
def test_peer_world1_matches_single_device(sg, golden, app):
    """world = 1: one partition holding every row, IPC-exported region, the
    device barrier with itself -- the reference's d1 run."""
    from paper_1911_09135_b200 import dist, native
    info = golden["runs"]["rmat12"][f"{app}/alb/d1"]
    g = _graph(sg, "rmat12")
    if app == "sssp":
        g = sg.attach_random_weights(g, 2)
    team = native.Team(0, 1, g.num_vertices)
    part = dist.partition(g, app, 0, 1)
    part2 = dist.partition(g, app, 0, 1, relabel=True)
    for pp in (part, part, part2):  # the team and the cached mirror masks are reused
        res = dist.run_app_peer(pp, app, sg.Scheduler("alb"), team=team)
        assert sg.engine.labels_sha256(res.labels) == info["labels_sha256"]
        assert [[r.frontier_size, r.active_edges()] for r in res.records] == \
            [x[:2] for x in info["per_round"]]


def test_peer_torchrun_two_processes():
    """Two processes (torchrun, gloo for the handle exchange) over CUDA IPC --
    one process per GPU when two are visible, otherwise both on this GPU."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29531", str(ROOT / "tests" / "peer_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    out = json.loads(line)
    assert out["world"] == 2
    for app, chk in out["apps"].items():
        assert chk["labels"] and chk["rounds"] and chk["comm_sent"] and chk["comm_broadcast"], \
            (app, chk)


def test_nccl_torchrun_world2():
    """The NCCL transport (sg_dist_run) with two processes, one GPU each --
    skipped on a one-GPU box (NCCL refuses two ranks on one device)."""
    from paper_1911_09135_b200 import native
    if native.device_count() < 2:
        pytest.skip("needs two GPUs (NCCL: one rank per device)")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29537", str(ROOT / "tests" / "nccl_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    out = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    for app, chk in out["apps"].items():
        assert all(chk.values()), (app, chk)
