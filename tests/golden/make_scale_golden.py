"""Golden records at the BASELINE configs' own scales, from the C oracle.

The numpy reference cannot run at RMAT-24..27 in reasonable time (SURVEY
Appendix C: hours, ~200 GB), so these records come from ``oracle/sg_oracle.c``
— the restatement pinned bit-for-bit to the unmodified reference by
tests/golden/golden.json (tests/test_oracle.py) and cross-checked against the
numpy oracle at RMAT <= 16.  Graphs: ``generate_rmat(scale, 16, 1, probs)``
(graph.py:274-298) rebuilt in C from the same PCG64 stream; sssp weights
``attach_random_weights(g, 2)`` (graph.py:301-305); kcore k = 2.

Each record: rounds, edges_processed, labels_sha256 (float64 labels, as
engine.report), the per-round (frontier_size, active_edges) log for the
frontier apps, and for pr the label sum / max and 64 sampled labels.

usage: python tests/golden/make_scale_golden.py KEY [KEY ...]   (see CONFIGS)
Appends/replaces entries in tests/golden/scale_golden.json.
"""
from __future__ import annotations

import gc
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle_c as C  # noqa: E402

OUT = Path(__file__).resolve().parent / "scale_golden.json"
SKEWED = (0.57, 0.19, 0.19, 0.05)
UNIFORM = (0.25, 0.25, 0.25, 0.25)
HEAVY = (0.8, 0.1, 0.05, 0.05)

# key -> (app, scale, probs)
CONFIGS = {
    "sssp/rmat24": ("sssp", 24, SKEWED),      # C2 (headline)
    "bfs/rmat24": ("bfs", 24, SKEWED),
    "cc/rmat24": ("cc", 24, SKEWED),
    "pr/rmat24": ("pr", 24, SKEWED),
    "kcore/rmat24": ("kcore", 24, SKEWED),
    "cc/rmat25": ("cc", 25, SKEWED),          # C3
    "pr/rmat25": ("pr", 25, SKEWED),          # C4 skewed
    "pr/uniform25": ("pr", 25, UNIFORM),      # C4 uniform
    "bfs/rmat27": ("bfs", 27, SKEWED),        # C5
    "kcore/rmat27": ("kcore", 27, SKEWED),    # C5
    "bfs/heavy24": ("bfs", 24, HEAVY),        # skew ablation
    "sssp/heavy24": ("sssp", 24, HEAVY),
    "cc/heavy24": ("cc", 24, HEAVY),
    "pr/heavy24": ("pr", 24, HEAVY),
    "kcore/heavy24": ("kcore", 24, HEAVY),
}


def sha(labels):
    return hashlib.sha256(np.ascontiguousarray(labels, dtype=np.float64).tobytes()).hexdigest()


def run_one(key):
    app, scale, probs = CONFIGS[key]
    thr = os.cpu_count() or 8
    t0 = time.time()
    off, tgt = C.rmat_csr(scale, 16, 1, probs, threads=thr)
    w = None
    if app == "sssp":
        rng = np.random.default_rng(np.random.PCG64(2))
        w = rng.integers(1, 65, size=len(tgt), dtype=np.int64).astype(np.float64)
    if app == "pr":
        coff, ctgt = C.transpose(off, tgt)
        view = (coff, ctgt, None, off, tgt)
    elif app in ("cc", "kcore"):
        soff, stgt = C.symmetrize(off, tgt, threads=thr)
        del off, tgt
        gc.collect()
        view = (soff, stgt, None, soff, stgt)
    else:
        view = (off, tgt, w, off, tgt)
    t_build = time.time() - t0
    t0 = time.time()
    lab, log, st = C.run(app, *view, threads=thr)
    t_run = time.time() - t0
    if st != 0:
        raise RuntimeError(f"{key}: oracle status {st}")
    rec = {"app": app, "scale": scale, "probs": list(probs), "edge_factor": 16, "seed": 1,
           "num_vertices": 1 << scale, "view_edges": int(len(view[1])),
           "rounds": int(len(log)), "edges_processed": int(log[:, 1].sum()),
           "labels_sha256": sha(lab), "oracle": "oracle/sg_oracle.c (OpenMP)",
           "threads": thr, "build_s": round(t_build, 1), "run_s": round(t_run, 1)}
    if app == "sssp":
        rec["weights"] = {"seed": 2, "low": 1, "high": 64}
    if app == "kcore":
        rec["k"] = 2
    if app == "pr":
        rec["damping"], rec["tol"] = 0.85, 1e-6
        rec["labels_sum"] = float(np.sum(lab))
        rec["labels_max"] = float(np.max(lab))
        idx = np.unique(np.concatenate([np.arange(32), np.linspace(0, len(lab) - 1, 32)
                                        .astype(np.int64)]))
        rec["sample_ids"] = idx.tolist()
        rec["sample_labels"] = [float(x).hex() for x in lab[idx]]
    else:
        rec["per_round"] = log.tolist()
        fin = lab[np.isfinite(lab)]
        rec["reached"] = int(len(fin))
    return rec


def main(keys):
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    for key in keys:
        rec = run_one(key)
        data[key] = rec
        OUT.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
        print(key, rec["rounds"], rec["edges_processed"], rec["labels_sha256"][:16],
              rec["run_s"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CONFIGS))
