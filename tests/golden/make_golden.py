"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run in the build container only (the reference is not present on GPU boxes):

    python tests/golden/make_golden.py

It imports ``simtgraph`` from /root/reference/pkg/src with the numpy kernel
backend forced (the shipped Cython module does not compile),
runs the reference's own public API (``engine.run_app`` / ``engine.report``,
``_kernels_py.lb_kernel`` / ``twc_kernel``) and writes:

* ``golden.json``   – per (graph, app, scheduler, devices) run: rounds,
  per-round frontier sizes / active edges / comm counters / launches,
  ``report()`` totals and ``labels_sha256``; plus the SPEC small fixtures.
* ``labels_small.npz`` – full float64 label arrays for the rmat10 / uniform10
  runs (small enough to commit).
* ``kernels_small.npz`` – kernel-level fixtures: inputs and outputs of the
  reference's ``lb_kernel`` / ``twc_kernel`` / ``vertex_kernel`` /
  ``edge_kernel`` on real rounds (the reference's plugin API).

Nothing under tests/ at run time reads /root/reference; only these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent

os.environ["SIMTGRAPH_KERNELS"] = "python"
sys.path.insert(0, REF)

from simtgraph import engine, graph as sgraph, schedulers, simt, _kernels_py  # noqa: E402
from simtgraph.apps import make_app  # noqa: E402

SKEWED = (0.57, 0.19, 0.19, 0.05)
UNIFORM = (0.25, 0.25, 0.25, 0.25)
APPS = ("bfs", "sssp", "cc", "pr", "kcore")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def graph_for(name: str):
    kind, scale = name[:-2], int(name[-2:])
    probs = SKEWED if kind == "rmat" else UNIFORM
    return sgraph.generate_rmat(scale, 16, 1, probs)


def run_one(g, gw, app, sched, devices, config=simt.KernelConfig()):
    graph = gw if app == "sssp" else g
    t0 = time.perf_counter()
    res = engine.run_app(graph, app, sched, config, devices=devices)
    dt = time.perf_counter() - t0
    rep = engine.report(res)
    rounds = []
    for rec in res.records:
        rounds.append([rec.frontier_size, rec.active_edges(), rec.comm_sent,
                       rec.comm_broadcast, rec.launches().get("lb", 0)])
    return res, {
        "rounds": rep["rounds"],
        "labels_sha256": rep["labels_sha256"],
        "edges_processed": rep["totals"]["edges_processed"],
        "search_memory_accesses": rep["totals"]["search_memory_accesses"],
        "inspect_degree_reads": rep["totals"]["inspect_degree_reads"],
        "comm_sent": rep["totals"]["comm_sent"],
        "comm_broadcast": rep["totals"]["comm_broadcast"],
        "kernel_launches": rep["totals"]["kernel_launches"],
        "worst_cta_cv": rep["load"]["worst_cta_cv"],
        "per_round": rounds,
        "ref_seconds": round(dt, 4),
    }


def spec_fixtures():
    """SPEC.md small examples, evaluated on the reference."""
    G = sgraph.Graph
    out = {}
    path = G.from_edges([0, 1], [1, 2], None, 3)
    out["path_bfs"] = engine.run_app(path, "bfs").labels.tolist()
    tri = G.from_edges([0, 0, 2], [1, 2, 1], [5, 1, 2], 3)
    out["triangle_sssp"] = engine.run_app(tri, "sssp").labels.tolist()
    two = G.from_edges([0, 2], [1, 3], None, 4)
    out["two_comp_cc"] = engine.run_app(two, "cc").labels.tolist()
    single = G(np.zeros(2, np.int64), np.zeros(0, np.int32), None, 1)
    out["single_pr"] = engine.run_app(single, "pr").labels.tolist()
    cyc = G.from_edges([0, 1], [1, 0], None, 2)
    out["two_cycle_pr"] = engine.run_app(cyc, "pr").labels.tolist()
    star = G.from_edges([0, 0, 0, 0, 1, 2, 3, 4], [1, 2, 3, 4, 0, 0, 0, 0], None, 5)
    out["star_pr"] = engine.run_app(star, "pr").labels.tolist()
    tri_u = G.from_edges([0, 1, 2], [1, 2, 0], None, 3)
    out["triangle_kcore2"] = engine.run_app(tri_u, "kcore", k=2).labels.tolist()
    ostar = G.from_edges([0, 0, 0], [1, 2, 3], None, 4)
    out["outstar_kcore2"] = engine.run_app(ostar, "kcore", k=2).labels.tolist()
    # unreachable vertices, self loops, duplicate edges, isolated vertices
    messy = G.from_edges([0, 0, 0, 1, 3, 3, 5], [0, 1, 1, 2, 4, 3, 5], [3, 2, 1, 7, 1, 1, 9], 7)
    for app in APPS:
        out[f"messy_{app}"] = engine.run_app(messy, app).labels.tolist()
    empty = G(np.zeros(5, np.int64), np.zeros(0, np.int32), None, 4)
    for app in APPS:
        out[f"empty4_{app}"] = engine.run_app(empty, app).labels.tolist()
    return out


def kernel_fixtures(g, gw):
    """Capture real lb/twc/vertex/edge kernel calls (the reference's plugin API)."""
    rec = {}
    cfg = simt.KernelConfig(4, 64, 32)  # small geometry so several passes occur
    idx = 0
    for app in ("bfs", "sssp", "cc", "pr", "kcore"):
        graph = gw if app == "sssp" else g
        run_graph = graph.symmetrized() if app in ("cc", "kcore") else graph
        a = make_app(app)
        a.setup(run_graph)
        view = schedulers.TraversalView.from_graph(run_graph, a.direction, unit_weights=a.needs_weights)
        frontier = a.initial_frontier()
        for rnd in range(3):
            if not len(frontier):
                break
            values = a.values
            aux = a.round_aux()
            degrees = view.degrees(frontier)
            for thr in (64, 1):
                huge, bins = schedulers.split_frontier(frontier, degrees, thr, cfg)
                for blocked in (0, 1):
                    if not len(huge):
                        continue
                    cum = np.cumsum(view.degrees(huge), dtype=np.int64)
                    if cum[-1] == 0:
                        continue
                    out = a.make_out()
                    pce = np.zeros(cfg.num_ctas, np.int64)
                    pwp = np.zeros(cfg.num_warps, np.int64)
                    acc = _kernels_py.lb_kernel(view.offsets, view.targets, view.weights, huge, cum,
                                                values, out, aux, a.opcode, blocked, cfg.num_ctas,
                                                cfg.threads_per_cta, cfg.warp_size, pce, pwp)
                    p = f"k{idx}_"
                    rec.update({p + "kind": np.array("lb"), p + "app": np.array(app),
                                p + "huge": huge, p + "cumulative": cum, p + "values": values.copy(),
                                p + "aux": aux.copy(), p + "opcode": np.array(a.opcode),
                                p + "blocked": np.array(blocked), p + "out": out,
                                p + "per_cta_edges": pce, p + "per_warp_paths": pwp,
                                p + "accesses": np.array(acc)})
                    idx += 1
                out = a.make_out()
                pce = np.zeros(cfg.num_ctas, np.int64)
                _kernels_py.twc_kernel(view.offsets, view.targets, view.weights, bins.small,
                                       bins.medium, bins.large, values, out, aux, a.opcode,
                                       cfg.num_ctas, cfg.threads_per_cta, cfg.warp_size, pce)
                p = f"k{idx}_"
                rec.update({p + "kind": np.array("twc"), p + "app": np.array(app),
                            p + "small": bins.small, p + "medium": bins.medium,
                            p + "large": bins.large, p + "values": values.copy(), p + "aux": aux.copy(),
                            p + "opcode": np.array(a.opcode), p + "out": out,
                            p + "per_cta_edges": pce})
                idx += 1
            for kind, fn in (("vertex", _kernels_py.vertex_kernel), ("edge", _kernels_py.edge_kernel)):
                out = a.make_out()
                pce = np.zeros(cfg.num_ctas, np.int64)
                fn(view.offsets, view.targets, view.weights, frontier, values, out, aux,
                   a.opcode, cfg.num_ctas, cfg.threads_per_cta, pce)
                p = f"k{idx}_"
                rec.update({p + "kind": np.array(kind), p + "app": np.array(app),
                            p + "frontier": frontier, p + "values": values.copy(), p + "aux": aux.copy(),
                            p + "opcode": np.array(a.opcode), p + "out": out,
                            p + "per_cta_edges": pce})
                idx += 1
            out = a.make_out()
            schedulers.run_round(schedulers.Scheduler("alb"), view, frontier,
                                 engine.RoundState(a.opcode, values, out, aux), cfg,
                                 simt.RoundMetrics(cfg))
            frontier, _ = a.end_round(out, frontier)
    rec["count"] = np.array(idx)
    rec["config"] = np.array([cfg.num_ctas, cfg.threads_per_cta, cfg.warp_size])
    return rec


def main():
    golden = {"numpy": np.__version__, "reference": "simtgraph 0.1.0 (numpy backend)",
              "edge_factor": 16, "seed": 1, "weights_seed": 2, "runs": {}}
    labels = {}
    plan = [
        ("rmat10", [("vertex", None), ("edge", None)], [1]),
        ("rmat10", [("alb", None), ("alb", 64), ("twc", None), ("lb", None)], [1, 2, 4]),
        ("uniform10", [("alb", None), ("alb", 64)], [1, 3]),
        ("rmat12", [("alb", None), ("alb", 256)], [1, 2, 4, 8]),
        ("rmat14", [("alb", None), ("alb", 1024)], [1]),
        ("rmat16", [("alb", None)], [1]),
        ("uniform16", [("alb", None)], [1]),
    ]
    for gname, scheds, devs in plan:
        g = graph_for(gname)
        gw = sgraph.attach_random_weights(g, 2)
        golden["runs"].setdefault(gname, {})["graph"] = {
            "num_vertices": g.num_vertices, "num_edges": g.num_edges,
            "offsets_sha256": sha(g.out_offsets), "targets_sha256": sha(g.out_targets),
            "weights_sha256": sha(gw.edge_weights),
            "csc_targets_sha256": sha(g.csc()[1]),
            "sym_targets_sha256": sha(g.symmetrized().out_targets),
            "sym_offsets_sha256": sha(g.symmetrized().out_offsets),
        }
        for app in APPS:
            for kind, thr in scheds:
                for d in devs:
                    key = f"{app}/{kind}" + (f"-t{thr}" if thr else "") + f"/d{d}"
                    sched = schedulers.Scheduler(kind, threshold=thr)
                    res, info = run_one(g, gw, app, sched, d)
                    golden["runs"][gname][key] = info
                    if gname.endswith("10") and kind == "alb" and thr is None and d == 1:
                        labels[f"{gname}_{app}"] = res.labels
                    print(gname, key, info["rounds"], info["edges_processed"],
                          info["labels_sha256"][:12], info["ref_seconds"], flush=True)
    golden["spec"] = spec_fixtures()
    (OUT / "golden.json").write_text(json.dumps(golden, indent=1, sort_keys=True) + "\n")
    np.savez_compressed(OUT / "labels_small.npz", **labels)
    g10 = graph_for("rmat10")
    np.savez_compressed(OUT / "kernels_small.npz",
                        **kernel_fixtures(g10, sgraph.attach_random_weights(g10, 2)))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
