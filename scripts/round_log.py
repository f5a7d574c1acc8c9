"""Print the device round log (frontier, edges, huge/large bins, updates) of one
app on rmat<scale>.  usage: python scripts/round_log.py app [scale] [threshold]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_1911_09135_b200 as sg  # noqa: E402

app = sys.argv[1]
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 24
thr = int(sys.argv[3]) if len(sys.argv) > 3 else bench.DEFAULT_THRESHOLD
gw, g = bench.make_graph_device(sg, app, scale, False)
_, p = bench.run_params(sg, app, "alb", thr, g.num_vertices)
_, log, ms = (gw if app == "sssp" else g).device().run(p)
print(f"{app} rmat{scale} t={thr}: {ms:.3f} ms")
for r in log:
    print({k: int(r[k]) for k in ("frontier_size", "active_edges", "huge_count", "huge_edges",
                                  "large_count", "large_edges", "updated")})
