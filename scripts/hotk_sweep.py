"""Hot-set size sweep of the relabeled store: SG_HOT_K=<K> python scripts/hotk_sweep.py
[scale] [apps]  (SG_HOT_K=off: the original numbering).  One JSON line per app."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_1911_09135_b200 as sg  # noqa: E402


def main():
    import torch
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    apps = sys.argv[2].split(",") if len(sys.argv) > 2 else ["sssp", "bfs", "cc", "pr", "kcore"]
    k = os.environ.get("SG_HOT_K", "default")  # default: the engine's per-app choice
    flags = 16 if k == "off" else 8
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    gw, g = bench.make_graph_device(sg, "sssp", scale, False)
    for app in apps:
        _, p = bench.run_params(sg, app, "alb", bench.DEFAULT_THRESHOLD, g.num_vertices)
        p.flags |= flags
        r = bench.device_steps(torch, (gw if app == "sssp" else g).device(), p, 5, 3, flush)
        print(json.dumps({"K": k, "scale": scale, "app": app, "gteps": round(r["gteps"], 2),
                          "ms": round(r["ms_per_step"], 3)}), flush=True)


if __name__ == "__main__":
    main()
