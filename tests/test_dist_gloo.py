"""CPU, world size 2 over gloo: the multi-GPU host path.

1. dist.share_nccl_id / dist.max_over_ranks / the IPC-handle all-gather
   (what bench.py / dist.run_app / dist.make_team use under torchrun) work
   across real processes;
2. the edge-cut exchange protocol of sg_dist.cu — local ALB round on the
   rank's row block, all-reduce(min) of the labels, sent-count before the
   exchange, diff of the owned range into the next local frontier, all-reduce
   (sum) of the round counters for quiescence — restated per rank with the
   oracle's kernels and gloo collectives, reproduces the reference's labels,
   per-round log and comm_sent / comm_broadcast for devices=2 exactly;
3. the same for the NVLink peer transport's protocol (sg_peer.cu: per-rank
   row storage, mirror -> owner min, owner -> mirror holders by mirror masks,
   labels gathered from the owners).
"""

from __future__ import annotations

import json
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _protocol(rank, world, app, dist, torch):
    from oracle import oracle_np as O
    from paper_1911_09135_b200.dist import partition_bounds
    off, tgt = O.rmat_csr(10)
    w = O.random_weights(len(tgt), 2) if app == "sssp" else None
    if app == "cc":
        off, tgt, _ = O.symmetrize(off, tgt)
    nv = len(off) - 1
    vw = (w.astype(np.float64) if w is not None else np.ones(len(tgt))) if app == "sssp" \
        else np.empty(0)
    op = {"bfs": O.OP_BFS, "sssp": O.OP_SSSP, "cc": O.OP_CC}[app]
    blocks, owner, mirror_count = O.edge_cut(off, tgt, world)
    assert blocks == partition_bounds(off, world)
    lo, hi = blocks[rank]
    if app == "cc":
        values = np.arange(nv, dtype=np.float64)
        local = np.arange(lo, hi, dtype=np.int64)
    else:
        values = np.full(nv, np.inf)
        values[0] = 0.0
        local = np.array([0], dtype=np.int64) if lo <= 0 < hi else np.empty(0, np.int64)
    log = []
    while True:
        out = values.copy()
        edges, lbl = 0, 0
        if len(local):
            edges, lbl = O.alb_round(off, tgt, vw, local, values, out, np.empty(0), op,
                                     84 * 256, 84, 256, 32)
        mine = np.ones(nv, bool)
        mine[lo:hi] = False
        sent = int(((out < values) & mine).sum())          # k_count_sent
        t = torch.from_numpy(out)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)          # ncclAllReduce(min)
        merged = t.numpy()
        own = np.arange(lo, hi)
        changed = own[merged[lo:hi] < values[lo:hi]]       # k_diff_owned
        bcast = int(mirror_count[changed].sum())
        acc = torch.tensor([len(local), edges, sent, bcast, len(changed)], dtype=torch.int64)
        dist.all_reduce(acc, op=dist.ReduceOp.SUM)        # ncclAllReduce(sum) of counters
        fs, ed, se, bc, nxt = (int(x) for x in acc)
        log.append([fs, ed, se, bc])
        values = merged.copy()
        local = changed.astype(np.int64)
        if nxt == 0:
            break
    return values, log


def _peer_protocol(rank, world, app, dist, torch):
    """The NVLink peer transport's protocol (sg_peer.cu) restated per rank:
    the rank stores only its rows, lowers its full-length label copy, sends
    each marked MIRROR to its owner (red.min; here a min-reduction that only
    carries marked entries), owners turn their changed rows into the next
    frontier and store each change into the ranks holding it as a mirror
    (mirror masks from the exchanged held bitmaps); counters are summed.
    Stale labels of vertices a rank neither owns nor holds are never read;
    the final labels are gathered from the owners."""
    from oracle import oracle_np as O
    from paper_1911_09135_b200.dist import partition_bounds
    off, tgt = O.rmat_csr(10)
    w = O.random_weights(len(tgt), 2) if app == "sssp" else None
    if app == "cc":
        off, tgt, _ = O.symmetrize(off, tgt)
    nv = len(off) - 1
    vw = (w.astype(np.float64) if w is not None else np.ones(len(tgt))) if app == "sssp" \
        else np.empty(0)
    op = {"bfs": O.OP_BFS, "sssp": O.OP_SSSP, "cc": O.OP_CC}[app]
    blocks = partition_bounds(off, world)
    lo, hi = blocks[rank]
    owner = np.zeros(nv, np.int64)
    for d, (a, b) in enumerate(blocks):
        owner[a:b] = d
    # this rank's partition: only rows [lo, hi) (offsets full length, rows outside empty)
    poff = np.clip(off, off[lo], off[hi]) - off[lo]
    ptgt = tgt[off[lo]:off[hi]]
    pw = vw[off[lo]:off[hi]] if len(vw) else vw
    held = np.zeros(nv, bool)                     # k_px_held
    held[ptgt[(ptgt < lo) | (ptgt >= hi)]] = True
    allheld = [torch.zeros(nv, dtype=torch.bool) for _ in range(world)]
    dist.all_gather(allheld, torch.from_numpy(held))
    holders = np.stack([h.numpy() for h in allheld])  # [rank, v]
    mcount = holders.sum(0)                       # popc(mask) == engine.py:84 mirror_count
    if app == "cc":
        lab = np.arange(nv, dtype=np.float64)
        local = np.arange(lo, hi, dtype=np.int64)
    else:
        lab = np.full(nv, np.inf)
        lab[0] = 0.0
        local = np.array([0], dtype=np.int64) if lo <= 0 < hi else np.empty(0, np.int64)
    inf = torch.full((nv,), float("inf"), dtype=torch.float64)
    log = []
    while True:
        out = lab.copy()
        edges = 0
        if len(local):
            edges, _ = O.alb_round(poff, ptgt, pw, local, lab, out, np.empty(0), op,
                                   84 * 256, 84, 256, 32)
        marked = out < lab                        # the bitmap (red.or on lowering)
        mirror = marked & (owner != rank)
        sent = int(mirror.sum())                  # k_px_reduce
        send = inf.clone()
        send[torch.from_numpy(mirror)] = torch.from_numpy(out[mirror])
        dist.all_reduce(send, op=dist.ReduceOp.MIN)   # remote red.min into the owners
        own = np.zeros(nv, bool)
        own[lo:hi] = True
        new = np.where(own, np.minimum(out, send.numpy()), out)
        changed = np.flatnonzero(own & (new < lab))   # k_px_compact
        bcast = int(mcount[changed].sum())
        upd = inf.clone()
        upd[torch.from_numpy(changed)] = torch.from_numpy(new[changed])
        dist.all_reduce(upd, op=dist.ReduceOp.MIN)    # owners' stores into mirror holders
        u = upd.numpy()
        mine = holders[rank] & np.isfinite(u) & ~own
        lab = new.copy()
        lab[mine] = np.minimum(lab[mine], u[mine])
        acc = torch.tensor([len(local), edges, sent, bcast, len(changed)], dtype=torch.int64)
        dist.all_reduce(acc, op=dist.ReduceOp.SUM)    # counter slots
        fs, ed, se, bc, nxt = (int(x) for x in acc)
        log.append([fs, ed, se, bc])
        local = changed.astype(np.int64)
        if nxt == 0:
            break
    final = inf.clone()
    final[lo:hi] = torch.from_numpy(lab[lo:hi])       # k_px_gather: each owner's block
    dist.all_reduce(final, op=dist.ReduceOp.MIN)
    return final.numpy(), log


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        sys.path.insert(0, str(ROOT))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1911_09135_b200 import dist as sgdist
        got_id = sgdist.share_nccl_id(dist, make_id=lambda: bytes(range(128)))
        mx = sgdist.max_over_ranks(dist, 1.5 + rank)
        res = {"id_ok": got_id == bytes(range(128)), "max": mx}
        import hashlib
        handles = sgdist._all_gather_bytes(dist, bytes([rank]) * 64)  # IPC handle exchange
        res["handles_ok"] = handles == [bytes([r]) * 64 for r in range(world)]
        for app in ("bfs", "sssp", "cc"):
            labels, log = _protocol(rank, world, app, dist, torch)
            res[app] = (hashlib.sha256(labels.tobytes()).hexdigest(), log)
            labels, log = _peer_protocol(rank, world, app, dist, torch)
            res["peer/" + app] = (hashlib.sha256(labels.tobytes()).hexdigest(), log)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(exc)}))


def test_edge_cut_protocol_world2_gloo(golden):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert "error" not in results[r], results[r].get("error")
        assert results[r]["id_ok"] and results[r]["max"] == 2.5
        assert results[r]["handles_ok"]
        for app in ("bfs", "sssp", "cc"):
            info = golden["runs"]["rmat10"][f"{app}/alb/d2"]
            for key in (app, "peer/" + app):
                sha, log = results[r][key]
                assert sha == info["labels_sha256"], (r, key)
                assert log == [x[:4] for x in info["per_round"]], (r, key)
