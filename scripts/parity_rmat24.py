"""Parity at the benchmark scale: every app on rmat24 (the bench's graph, run
twice so the second run takes the relabeled store) against the C oracle
(OpenMP) -- bit-identical labels and round logs (pr: 1e-7, rounds +-1).
usage: python scripts/parity_rmat24.py [scale]  -> one JSON line per app"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1911_09135_b200 as sg  # noqa: E402
from oracle import oracle_c as C  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    g = sg.generate_rmat(scale, 16, 1)
    gw = sg.attach_random_weights(g, 2)
    off, tgt, w = g.out_offsets, g.out_targets, gw.edge_weights
    for app in ("bfs", "sssp", "cc", "kcore", "pr"):
        t0 = time.time()
        lab, log, st = C.run(app, *C.prepare(off, tgt, w if app == "sssp" else None, app),
                             threads=os.cpu_count() or 8)
        t_cpu = time.time() - t0
        out = {"app": app, "scale": scale, "oracle_s": round(t_cpu, 1), "runs": []}
        for run in range(2):
            res = sg.run_app(gw if app == "sssp" else g, app, sg.Scheduler("alb"))
            rounds = [[r.frontier_size, r.active_edges()] for r in res.records]
            if app == "pr":
                ok = abs(len(rounds) - len(log)) <= 1 and \
                    float(np.max(np.abs(res.labels - lab))) <= 1e-7
                err = float(np.max(np.abs(res.labels - lab)))
                out["runs"].append({"ok": bool(ok), "max_abs": err, "rounds": len(rounds),
                                    "oracle_rounds": len(log)})
            else:
                ok = rounds == log.tolist() and bool(np.array_equal(res.labels, lab))
                out["runs"].append({"ok": bool(ok), "rounds": len(rounds)})
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
