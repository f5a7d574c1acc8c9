"""SGB1 load into HBM: sg_graph_load_sgb1 (path) vs the reference's host parse
(numpy frombuffer + Graph validation, graph.py:159-177) followed by the upload.
The file is written first, so both read from the page cache.
usage: python scripts/io_bench.py [scale]   -> one JSON line"""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_1911_09135_b200 as sg  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    g = sg.attach_random_weights(sg.generate_rmat(scale, 16, 1), 2)
    fd, path = tempfile.mkstemp(suffix=".sgb")
    os.close(fd)
    try:
        g.save_binary(path)
        size = os.path.getsize(path)
        dev = []
        for _ in range(3):
            t0 = time.perf_counter()
            h = sg.Graph.load_binary(path)
            h.device().info()
            dev.append(time.perf_counter() - t0)
            del h
        host = []
        for _ in range(2):
            t0 = time.perf_counter()
            with open(path, "rb") as f:
                h = sg.Graph.load_binary(f)
            h.device()
            host.append(time.perf_counter() - t0)
        h = sg.Graph.load_binary(path)
        same = bool(np.array_equal(h.edge_weights, g.edge_weights)
                    and np.array_equal(h.out_targets, g.out_targets))
        print(json.dumps({"scale": scale, "file_bytes": size,
                          "device_loader_s": round(min(dev), 4),
                          "device_loader_GBps": round(size / min(dev) / 1e9, 2),
                          "host_parse_upload_s": round(min(host), 4),
                          "host_parse_upload_GBps": round(size / min(host) / 1e9, 2),
                          "arrays_equal": same, "nproc": os.cpu_count()}))
    finally:
        os.unlink(path)


if __name__ == "__main__":
    main()
