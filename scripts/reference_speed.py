"""Times the UNMODIFIED reference (numpy backend, single thread) on rmat16/18/20 in
the build container -- context for the C-port baselines; needs /root/reference
(absent on the GPU box).  usage: python scripts/reference_speed.py"""
import sys, time, json, os
sys.path.insert(0, '/root/reference/pkg/src')
import simtgraph as S
from simtgraph import engine, graph, schedulers, simt
out = []
for scale in (16, 18, 20):
    g = graph.generate_rmat(scale, 16, 1)
    gw = graph.attach_random_weights(g, 2)
    for app in ("bfs", "sssp"):
        gg = gw if app == "sssp" else g
        t0 = time.perf_counter()
        res = engine.run_app(gg, app, schedulers.Scheduler("alb"), simt.KernelConfig(), 1)
        dt = time.perf_counter() - t0
        e = engine.report(res)["totals"]["edges_processed"]
        out.append({"scale": scale, "app": app, "seconds": round(dt, 3), "edges_processed": e,
                    "gteps": e / dt / 1e9})
        print(json.dumps(out[-1]), flush=True)
