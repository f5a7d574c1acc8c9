"""pr exactness + speed probe: golden shas (rmat10..16, uniform), rmat24 vs the
scale golden on both layouts, per-run times.  JSON lines on stdout."""
import json, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1911_09135_b200 as sg

gold = json.loads((ROOT / "tests/golden/golden.json").read_text())
for gname, runs in gold["runs"].items():
    kind, scale = gname[:-2], int(gname[-2:])
    g = sg.generate_rmat(scale, 16, 1, sg.graph.RMAT_SKEWED if kind == "rmat" else sg.graph.RMAT_UNIFORM)
    for key, info in runs.items():
        if not key.startswith("pr/"):
            continue
        _, sched, dev = key.split("/")
        k = sched.split("-")[0]
        thr = int(sched.split("-t")[1]) if "-t" in sched else None
        res = sg.run_app(g, "pr", sg.Scheduler(k, threshold=thr), devices=int(dev[1:]))
        print(json.dumps({"run": f"{gname}/{key}", "sha_ok": sg.engine.labels_sha256(res.labels) == info["labels_sha256"],
                          "rounds": len(res.records), "want": info["rounds"]}), flush=True)
sc = json.loads((ROOT / "tests/golden/scale_golden.json").read_text())
scales = [int(x) for x in sys.argv[1:]] or [24]
for s in scales:
    key = f"pr/rmat{s}"
    if key not in sc:
        continue
    g = sg.generate_rmat(s, 16, 1)
    for run in range(3):
        t = time.perf_counter()
        res = sg.run_app(g, "pr")
        dt = time.perf_counter() - t
        info = sc[key]
        print(json.dumps({"run": f"{key} run{run}", "sha_ok": sg.engine.labels_sha256(res.labels) == info["labels_sha256"],
                          "rounds": len(res.records), "want": info["rounds"], "wall_s": round(dt, 3),
                          "device_ms": res.device_ms,
                          "max_abs_vs_sample": float(np.max(np.abs(res.labels[info["sample_ids"]] - np.array([float.fromhex(x) for x in info["sample_labels"]]))))}), flush=True)
