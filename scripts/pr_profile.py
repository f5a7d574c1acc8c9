"""Per-kernel times of one pr run (profiled: CUDA events around every kernel)
and plain run times, for the current build / env (SG_EXACT_HS ...).
usage: python scripts/pr_profile.py SCALE [uniform]"""
import json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1911_09135_b200 as sg
from paper_1911_09135_b200 import native
import bench

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
uni = len(sys.argv) > 2 and sys.argv[2] == "uniform"
g, _ = bench.make_graph_device(sg, "pr", scale, uni)
dev = g.device()
nv, ne, _ = dev.info()
sched, params = bench.run_params(sg, "pr", "alb", None, nv, False)
ms = []
for i in range(4):
    lab, log, t = dev.run(params)
    ms.append(t)
_, plog, pms, kernels = dev.run(params, profile=True)
import os
print(json.dumps({"scale": scale, "uniform": uni, "hs": os.environ.get("SG_EXACT_HS", "2048 (default)"),
                  "rounds": len(log), "ms_runs": [round(x, 2) for x in ms],
                  "gteps": round(int(log["active_edges"].sum()) / (min(ms[1:]) / 1e3) / 1e9, 1),
                  "kernels": {k: [v[0], round(v[1], 3)] for k, v in kernels.items()}}), flush=True)
