"""torchrun worker for tests/test_gpu_peer.py (not collected by pytest): every
rank cuts its partition of rmat12, joins the NVLink peer team and runs the
five apps; rank 0 checks labels, round log and comm counters against the
reference's devices=WORLD goldens and prints one JSON line.  With fewer GPUs
than ranks, ranks share a GPU (IPC mappings of the same device)."""

import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch.distributed as tdist

    import paper_1911_09135_b200 as sg
    from paper_1911_09135_b200 import dist

    rank, _, world = dist.env()
    dist.init_device()
    tdist.init_process_group("gloo", init_method="env://")
    golden = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
    g = sg.generate_rmat(12, 16, 1)
    gw = sg.attach_random_weights(g, 2)
    team = dist.make_team(tdist, g.num_vertices)
    result = {}
    for app, relabel in [(a, r) for r in (False, True)
                         for a in ("bfs", "sssp", "cc", "pr", "kcore")]:
        part = dist.partition(gw if app == "sssp" else g, app, rank, world, relabel=relabel)
        res = dist.run_app_peer(part, app, sg.Scheduler("alb"), team=team)
        info = golden["runs"]["rmat12"][f"{app}/alb/d{world}"]
        rounds = [[r.frontier_size, r.active_edges()] for r in res.records]
        comm = [[r.comm_sent, r.comm_broadcast] for r in res.records]
        result[f"{app}{'/relabel' if relabel else ''}"] = {
            "labels": sg.engine.labels_sha256(res.labels) == info["labels_sha256"],
            "rounds": rounds == [x[:2] for x in info["per_round"]],
            "comm_sent": [c[0] for c in comm] == [x[2] for x in info["per_round"]],
            "comm_broadcast": [c[1] for c in comm] == [x[3] for x in info["per_round"]],
            "local_edges": part.local_edges,
            "view_edges": part.view_edges,
        }
    team.close()
    tdist.barrier()
    if rank == 0:
        print(json.dumps({"world": world, "apps": result}))
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
