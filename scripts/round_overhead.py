"""Fixed per-round cost of the device BSP loop: BFS / SSSP on a path graph
(one vertex and one edge per round).  usage: python scripts/round_overhead.py [n]"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_1911_09135_b200 as sg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
g = sg.Graph.from_edges(np.arange(n - 1), np.arange(1, n), np.ones(n - 1, np.int64), n)
for app in ("bfs", "sssp"):
    _, p = bench.run_params(sg, app, "alb", bench.DEFAULT_THRESHOLD, n)
    d = g.device()
    for _ in range(3):
        labels, log, ms = d.run(p)
    best = min(d.run(p)[2] for _ in range(5))
    print(f"{app}: {len(log)} rounds, {best:.3f} ms, {1e3 * best / len(log):.2f} us/round")
