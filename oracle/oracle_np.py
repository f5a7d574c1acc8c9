"""CPU oracle (numpy) for the ALB BSP hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It restates the reference
``simtgraph`` algorithm (numpy backend; /root/reference/pkg/src/simtgraph)
so parity can be checked on machines where the reference is absent.

Pinned against ``tests/golden/*`` (produced by running the unmodified
reference, see ``tests/golden/make_golden.py``): every run-level sha256,
round count and per-round (frontier, active edges, comm) log, and every
kernel-level fixture (``out``, ``per_cta_edges``, ``per_warp_paths``,
search accesses) — see ``tests/test_oracle.py``.

Third-party arithmetic: numpy 2.3.5 (``PCG64`` + ``Generator.random`` /
``Generator.integers``, stable ``argsort``, ``ufunc.at``); the graph identity
of ``generate_rmat`` is pinned to that numpy version.
"""

from __future__ import annotations

import math

import numpy as np

OP_BFS, OP_SSSP, OP_CC, OP_PULL_ADD = 0, 1, 2, 3  # _kernels_py.py:26-29
SKEWED = (0.57, 0.19, 0.19, 0.05)  # graph.py:26


# ----------------------------------------------------------------------------
# graph construction (graph.py)
# ----------------------------------------------------------------------------

def csr_from_pairs(src, dst, weights=None, nv=None):
    """Stable counting sort by source (graph.py:63-76)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    if nv is None:
        nv = int(max(src.max(), dst.max())) + 1 if len(src) else 0
    off = np.zeros(nv + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=nv), out=off[1:])
    perm = np.argsort(src, kind="stable")
    tgt = dst[perm].astype(np.int32)
    w = None if weights is None else np.asarray(weights, dtype=np.int64)[perm]
    return off, tgt, w


def rmat_pairs(scale, edge_factor=16, seed=1, probs=SKEWED):
    """Edge (src, dst) stream of generate_rmat (graph.py:274-298).

    Level l, edge i consumes PCG64 draw number l*E+i via Generator.random.
    """
    nv = 1 << scale
    ne = edge_factor * nv
    gen = np.random.default_rng(np.random.PCG64(seed))
    thresholds = np.cumsum(np.asarray(probs, dtype=np.float64))[:3]
    src = np.zeros(ne, dtype=np.int64)
    dst = np.zeros(ne, dtype=np.int64)
    for _level in range(scale):
        q = np.searchsorted(thresholds, gen.random(ne), side="right")
        src = (src << 1) | (q >> 1)
        dst = (dst << 1) | (q & 1)
    return src, dst, nv


def rmat_csr(scale, edge_factor=16, seed=1, probs=SKEWED):
    src, dst, nv = rmat_pairs(scale, edge_factor, seed, probs)
    off, tgt, _ = csr_from_pairs(src, dst, None, nv)
    return off, tgt


def random_weights(ne, seed, low=1, high=64):
    """attach_random_weights (graph.py:301-305)."""
    return np.random.default_rng(np.random.PCG64(seed)).integers(low, high + 1, size=ne, dtype=np.int64)


def row_ids(off):
    return np.repeat(np.arange(len(off) - 1, dtype=np.int64), np.diff(off))


def transpose(off, tgt, w=None):
    """CSC by stable sort on target (graph.py:95-113)."""
    nv = len(off) - 1
    in_off = np.zeros(nv + 1, dtype=np.int64)
    np.cumsum(np.bincount(tgt, minlength=nv), out=in_off[1:])
    perm = np.argsort(tgt, kind="stable")
    in_tgt = np.ascontiguousarray(row_ids(off).astype(np.int32)[perm])
    in_w = None if w is None else w[perm]
    return in_off, in_tgt, in_w


def symmetrize(off, tgt, w=None):
    """Edge multiset union with its reverse (graph.py:115-128)."""
    s = row_ids(off)
    d = tgt.astype(np.int64)
    ww = None if w is None else np.concatenate([w, w])
    return csr_from_pairs(np.concatenate([s, d]), np.concatenate([d, s]), ww, len(off) - 1)


# ----------------------------------------------------------------------------
# kernels (_kernels_py.py) — the reference's plugin API, with its counters
# ----------------------------------------------------------------------------

def search_depths(n):
    """Bisection probe count per landing segment (_kernels_py.py:34-56)."""
    d = np.zeros(n, dtype=np.int64)
    todo = [(0, n - 1, 0)]
    while todo:
        lo, hi, k = todo.pop()
        if lo == hi:
            d[lo] = k
            continue
        m = (lo + hi) // 2
        todo += [(lo, m, k + 1), (m + 1, hi, k + 1)]
    return d


def ranges(starts, lens):
    """Concatenated arange blocks (_kernels_py.py:59-66)."""
    n = int(lens.sum())
    if n == 0:
        return np.empty(0, dtype=np.int64)
    blk = np.repeat(np.arange(len(lens)), lens)
    first = np.cumsum(lens) - lens
    return starts[blk] + np.arange(n, dtype=np.int64) - first[blk]


def apply_edges(op, rows, eidx, tgt, w, values, out, aux):
    """Operator over edges in array order (_kernels_py.py:69-85)."""
    if len(eidx) == 0:
        return
    if op == OP_PULL_ADD:
        np.add.at(out, rows, aux[tgt[eidx]])
        return
    if op == OP_BFS:
        prop = values[rows] + 1.0
    elif op == OP_SSSP:
        prop = values[rows] + w[eidx]
    elif op == OP_CC:
        prop = values[rows]
    else:
        raise ValueError(f"unknown opcode {op}")
    np.minimum.at(out, tgt[eidx], prop)


def vertex_kernel(off, tgt, w, frontier, values, out, aux, op, ctas, tpb, pce):
    """_kernels_py.py:88-97."""
    deg = off[frontier + 1] - off[frontier]
    np.add.at(pce, (np.arange(len(frontier)) % (ctas * tpb)) // tpb, deg)
    apply_edges(op, np.repeat(frontier, deg), ranges(off[frontier], deg), tgt, w, values, out, aux)


def edge_kernel(off, tgt, w, frontier, values, out, aux, op, ctas, tpb, pce):
    """_kernels_py.py:100-117."""
    deg = off[frontier + 1] - off[frontier]
    eidx = ranges(off[frontier], deg)
    m = len(eidx)
    if m == 0:
        return
    per = -(-m // (ctas * tpb))
    pce += np.bincount((np.arange(m) // per) // tpb, minlength=ctas)
    apply_edges(op, np.repeat(frontier, deg), eidx, tgt, w, values, out, aux)


def twc_kernel(off, tgt, w, small, medium, large, values, out, aux, op, ctas, tpb, ws, pce):
    """_kernels_py.py:120-150 (thread / warp / CTA attribution)."""
    threads = ctas * tpb
    rows, eidx = [], []
    for ids, cta_of in ((small, lambda i: (i % threads) // tpb),
                        (medium, lambda i: (i % (threads // ws)) // (tpb // ws)),
                        (large, lambda i: i % ctas)):
        if not len(ids):
            continue
        deg = off[ids + 1] - off[ids]
        np.add.at(pce, cta_of(np.arange(len(ids))), deg)
        rows.append(np.repeat(ids, deg))
        eidx.append(ranges(off[ids], deg))
    if rows:
        apply_edges(op, np.concatenate(rows), np.concatenate(eidx), tgt, w, values, out, aux)


def lb_kernel(off, tgt, w, huge, cum, values, out, aux, op, blocked, ctas, tpb, ws, pce, pwp):
    """_kernels_py.py:153-201: owner search + warp-pass search accounting."""
    e = int(cum[-1])
    threads = ctas * tpb
    nwarps = threads // ws
    if blocked:
        per = -(-e // threads)
        pas = np.repeat(np.arange(per, dtype=np.int64), threads)
        tid = np.tile(np.arange(threads, dtype=np.int64), per)
        g = tid * per + pas
        keep = g < e
        g, tid, pas = g[keep], tid[keep], pas[keep]
    else:
        g = np.arange(e, dtype=np.int64)
        tid = g % threads
        pas = g // threads
    key = pas * nwarps + tid // ws
    own = np.searchsorted(cum, g, side="right")
    base = np.where(own > 0, cum[own - 1], 0)
    rows = huge[own]
    pce += np.bincount(tid // tpb, minlength=ctas)
    apply_edges(op, rows, off[rows] + (g - base), tgt, w, values, out, aux)
    # one search is charged per (warp, pass) group and distinct owner
    grp = np.ones(len(g), dtype=bool)
    grp[1:] = key[1:] != key[:-1]
    newp = grp.copy()
    newp[1:] |= own[1:] != own[:-1]
    accesses = int(search_depths(len(cum))[own[newp]].sum())
    seg = np.cumsum(grp) - 1
    np.maximum.at(pwp, key[grp] % nwarps, np.bincount(seg[newp]))
    return accesses


# ----------------------------------------------------------------------------
# BSP engine + apps (engine.py, apps.py, schedulers.py)
# ----------------------------------------------------------------------------

class Round:
    __slots__ = ("frontier_size", "active_edges", "comm_sent", "comm_broadcast", "lb_launches",
                 "pce", "accesses", "launches")

    def __init__(self, n):
        self.frontier_size = n
        self.active_edges = 0
        self.comm_sent = 0
        self.comm_broadcast = 0
        self.lb_launches = 0
        self.pce = []          # per-device per-CTA edge arrays (simt.py:73-90)
        self.accesses = 0      # modeled search accesses (lb kernel)
        self.launches = {}     # kernel name -> launches (schedulers.py:252-298)

    def as_list(self):
        return [self.frontier_size, self.active_edges, self.comm_sent, self.comm_broadcast,
                self.lb_launches]

    def cta_cv(self):
        e = np.concatenate(self.pce) if self.pce else np.zeros(0)
        m = e.mean() if len(e) else 0.0
        return float(e.std() / m) if m > 0 else 0.0


def edge_cut(off, tgt, devices):
    """Edge-balanced contiguous row blocks + mirror counts (engine.py:64-85)."""
    nv = len(off) - 1
    total = int(off[-1])
    cuts = [0]
    for k in range(1, devices):
        c = int(np.searchsorted(off, round(k * total / devices), side="left"))
        cuts.append(max(c, cuts[-1]))
    cuts.append(nv)
    blocks = [(cuts[d], cuts[d + 1]) for d in range(devices)]
    owner = np.zeros(nv, dtype=np.int64)
    mirror_count = np.zeros(nv, dtype=np.int64)
    for d, (a, b) in enumerate(blocks):
        owner[a:b] = d
        t = tgt[off[a]:off[b]]
        mirror_count[np.unique(t[(t < a) | (t >= b)]).astype(np.int64)] += 1
    return blocks, owner, mirror_count


def alb_round(off, tgt, w, frontier, values, out, aux, op, threshold, ctas, tpb, ws,
              kind="alb", blocked=False, K=None, rec=None):
    """schedulers.run_round for every scheduler kind (schedulers.py:252-298).

    ``K`` is a module with the plugin's four kernels (default: this file's
    restatement; tests pass ``paper_1911_09135_b200.cuda_backend``); ``rec``
    collects per-CTA edges, search accesses and launches like RoundMetrics."""
    import sys
    K = K or sys.modules[__name__]
    pce = np.zeros(ctas, dtype=np.int64)
    pwp = np.zeros(ctas * tpb // ws, dtype=np.int64)
    lb = 0
    acc = 0
    launches = {}

    def launch(name):
        launches[name] = launches.get(name, 0) + 1

    deg = off[frontier + 1] - off[frontier]
    if kind in ("vertex", "edge"):
        launch(kind)
        (K.vertex_kernel if kind == "vertex" else K.edge_kernel)(
            off, tgt, w, frontier, values, out, aux, op, ctas, tpb, pce)
    elif kind == "lb":
        cum = np.cumsum(deg, dtype=np.int64)
        if len(cum) and cum[-1] > 0:
            launch("lb")
            acc += int(K.lb_kernel(off, tgt, w, frontier, cum, values, out, aux, op, blocked,
                                   ctas, tpb, ws, pce, pwp))
            lb = 1
    else:
        launch("inspect")
        if kind == "alb":
            big = deg >= threshold
            huge, rest, rdeg = frontier[big], frontier[~big], deg[~big]
            if len(huge):
                cum = np.cumsum(off[huge + 1] - off[huge], dtype=np.int64)
                launch("lb")
                acc += int(K.lb_kernel(off, tgt, w, huge, cum, values, out, aux, op, blocked,
                                       ctas, tpb, ws, pce, pwp))
                lb = 1
        else:
            rest, rdeg = frontier, deg
        small = rdeg < ws
        large = rdeg >= tpb
        launch("twc")
        K.twc_kernel(off, tgt, w, rest[small], rest[~small & ~large], rest[large], values, out,
                     aux, op, ctas, tpb, ws, pce)
    if rec is not None:
        rec.pce.append(pce)
        rec.accesses += acc
        for k, n in launches.items():
            rec.launches[k] = rec.launches.get(k, 0) + n
    return int(pce.sum()), lb


def run(off, tgt, weights, app, *, source=0, k=2, damping=0.85, tol=1e-6, kind="alb",
        threshold=None, blocked=False, ctas=84, tpb=256, ws=32, devices=1, max_rounds=None,
        directed_off=None, directed_tgt=None, K=None):
    """engine.run for one app over the graph ``(off, tgt, weights)``.

    For cc / kcore pass the SYMMETRIZED graph (engine.py:195).  For pr pass the
    directed CSR; the CSC pull view is built here (schedulers.py:100-113).
    Returns (labels float64, [Round]).  Raises RuntimeError on non-convergence
    (engine.py:206-209 raises ConvergenceError).
    """
    nv = len(off) - 1
    if threshold is None:
        threshold = ctas * tpb  # schedulers.py:58-60
    threshold = max(1, int(threshold))  # worklist.py:122-128
    if app in ("bfs", "sssp"):
        if not 0 <= source < nv:
            raise ValueError(f"source {source} outside graph")
        op = OP_BFS if app == "bfs" else OP_SSSP
        voff, vtgt = off, tgt
        if app == "sssp":
            vw = (weights.astype(np.float64) if weights is not None
                  else np.ones(len(tgt), dtype=np.float64))
        else:
            vw = None if weights is None else weights.astype(np.float64)
        values = np.full(nv, np.inf)
        values[source] = 0.0
        frontier = np.array([source], dtype=np.int64)
        merge = "min"
    elif app == "cc":
        op, voff, vtgt = OP_CC, off, tgt
        vw = None if weights is None else weights.astype(np.float64)
        values = np.arange(nv, dtype=np.float64)
        frontier = np.arange(nv, dtype=np.int64)
        merge = "min"
    elif app == "pr":
        op = OP_PULL_ADD
        voff, vtgt, _ = transpose(off, tgt)
        vw = None
        outdeg = np.diff(off)
        inv = np.zeros(nv, dtype=np.float64)
        inv[outdeg > 0] = 1.0 / outdeg[outdeg > 0]
        values = np.full(nv, 1.0 - damping)
        if len(tgt):
            gain = np.bincount(tgt, weights=inv[row_ids(off)], minlength=nv)
            worst = damping * gain.max()
        else:
            worst = 0.0
        eps_stop = tol / max(1.0, worst)  # apps.py:163-171
        frontier = np.arange(nv, dtype=np.int64)
        merge = "add"
    elif app == "kcore":
        op = OP_PULL_ADD
        voff, vtgt, _ = transpose(off, tgt)
        vw = None
        values = np.ones(nv, dtype=np.float64)
        frontier = np.arange(nv, dtype=np.int64)
        merge = "add"
    else:
        raise ValueError(f"unknown app {app!r}")
    if vw is None:
        vw = np.empty(0, dtype=np.float64)
    blocks, owner, mirror_count = edge_cut(voff, vtgt, devices)
    if max_rounds is None:
        max_rounds = 10 * max(nv, 1) + 256  # engine.py:199-202
    log = []
    while len(frontier):
        if len(log) >= max_rounds:
            raise RuntimeError(f"{app} did not converge within {max_rounds} rounds")
        if app == "pr":
            aux = values * inv
        elif app == "kcore":
            aux = values
        else:
            aux = np.empty(0, dtype=np.float64)
        rec = Round(len(frontier))
        outs = []
        for (a, b) in blocks:
            out = values.copy() if merge == "min" else np.zeros(nv, dtype=np.float64)
            local = frontier[np.searchsorted(frontier, a):np.searchsorted(frontier, b)]
            if len(local):
                m, lb = alb_round(voff, vtgt, vw, local, values, out, aux, op, threshold,
                                  ctas, tpb, ws, kind, blocked, K, rec)
                rec.active_edges += m
                rec.lb_launches += lb
            outs.append(out)
        merged = outs[0].copy()
        if devices > 1:
            base = values if merge == "min" else np.zeros(nv)
            for d, o in enumerate(outs):
                rec.comm_sent += int(((o != base) & (owner != d)).sum())
            for o in outs[1:]:
                if merge == "min":
                    np.minimum(merged, o, out=merged)
                else:
                    merged += o
        before = values.copy()
        if merge == "min":
            frontier = np.flatnonzero(merged < values)
            values = merged
        elif app == "pr":
            new = (1.0 - damping) + damping * merged
            delta = np.abs(new - values).max() if nv else 0.0
            values = new
            frontier = (np.empty(0, dtype=np.int64) if delta <= eps_stop
                        else np.arange(nv, dtype=np.int64))
        else:  # kcore (apps.py:220-232)
            dying = frontier[merged[frontier] < k]
            if len(dying):
                values[dying] = 0.0
                nb = np.unique(np.concatenate([tgt[off[v]:off[v + 1]] for v in dying.tolist()]))
                frontier = nb[values[nb] > 0.0].astype(np.int64)
            else:
                frontier = np.empty(0, dtype=np.int64)
        if devices > 1:
            rec.comm_broadcast = int(mirror_count[values != before].sum())
        log.append(rec)
    return values, log


def run_graph(off, tgt, weights, app, **kw):
    """Convenience: symmetrize for cc / kcore as engine.run does (engine.py:195)."""
    if app in ("cc", "kcore"):
        off, tgt, weights = symmetrize(off, tgt, weights)
    return run(off, tgt, weights, app, **kw)


def labels_sha256(labels):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(labels, dtype=np.float64).tobytes()).hexdigest()


def gteps(edges, seconds):
    return edges / seconds / 1e9 if seconds > 0 else math.inf
