"""Huge-vertex threshold sweep (the reference CLI's sweep-threshold, cli.py:239-290;
the paper's threshold sensitivity): ALB GTEPS on rmat24 per threshold, labels
checked equal across thresholds.  usage: python scripts/threshold_sweep.py [scale] [apps]"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_1911_09135_b200 as sg  # noqa: E402

THRESHOLDS = [32, 256, 1024, 4096, 21504, 65536, 262144, None]  # None: TWC-only (inf)


def main():
    import torch
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    apps = sys.argv[2].split(",") if len(sys.argv) > 2 else ["sssp", "bfs", "cc", "kcore", "pr"]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    gw, g = bench.make_graph_device(sg, "sssp", scale, False)
    for app in apps:
        dev = (gw if app == "sssp" else g).device()
        row, ref = {}, None
        for t in THRESHOLDS:
            kind = "twc" if t is None else "alb"
            _, p = bench.run_params(sg, app, kind, t or 0, g.num_vertices)
            r = bench.device_steps(torch, dev, p, 3 if app == "pr" else 5, 3, flush)
            labels, _, _ = dev.run(p)
            if ref is None:
                ref = labels
            same = bool(np.array_equal(labels, ref)) if app != "pr" else \
                bool(np.max(np.abs(labels - ref)) <= 1e-7)
            row["inf" if t is None else str(t)] = {"gteps": round(r["gteps"], 1), "labels_equal": same}
        print(json.dumps({"app": app, "scale": scale, "sweep": row}), flush=True)


if __name__ == "__main__":
    main()
