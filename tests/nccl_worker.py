"""torchrun worker for tests/test_gpu_peer.py::test_nccl_torchrun_world2 (not
collected by pytest): every rank runs the five apps through the NCCL edge-cut
transport (sg_dist_run, one GPU per rank) and rank 0 prints one JSON line with
the label / round-log / comm-counter checks against the reference's
devices=WORLD goldens."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import torch.distributed as tdist

    import paper_1911_09135_b200 as sg
    from paper_1911_09135_b200 import dist

    rank, local, world = dist.env()
    dev = dist.init_device()
    tdist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    golden = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
    g = sg.generate_rmat(12, 16, 1)
    gw = sg.attach_random_weights(g, 2)
    nccl_id = dist.share_nccl_id(tdist)
    result = {}
    for app in ("bfs", "sssp", "cc", "pr", "kcore"):
        res = dist.run_app(gw if app == "sssp" else g, app, sg.Scheduler("alb"), rank=rank,
                           world=world, nccl_id=nccl_id)
        info = golden["runs"]["rmat12"][f"{app}/alb/d{world}"]
        result[app] = {
            "labels": sg.engine.labels_sha256(res.labels) == info["labels_sha256"],
            "rounds": [[r.frontier_size, r.active_edges()] for r in res.records]
            == [x[:2] for x in info["per_round"]],
            "comm_sent": [r.comm_sent for r in res.records] == [x[2] for x in info["per_round"]],
        }
    dist.release()
    tdist.barrier()
    if rank == 0:
        print(json.dumps({"world": world, "apps": result}))
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
