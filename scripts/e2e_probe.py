"""Break the bench's e2e step (host CSR -> sg_graph_create -> sg_run -> labels)
into its parts on the GPU box (diagnostics, not a bench line)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1911_09135_b200 as sg  # noqa: E402
from paper_1911_09135_b200 import native  # noqa: E402

app = sys.argv[1] if len(sys.argv) > 1 else "sssp"
g = sg.generate_rmat(24, 16, 1)
g = sg.attach_random_weights(g, 2) if app == "sssp" else g
dev = g.device()
nv, ne, _ = dev.info()
params = sg.engine.device_params(sg.apps.make_app(app), sg.Scheduler("alb"), sg.KernelConfig(), 1,
                                  10 * nv + 256)
off, tgt, w = dev.download(0, weights=(app == "sssp"))
pin = lambda x: torch.from_numpy(x).pin_memory().numpy() if x is not None else None
off_p, tgt_p, w_p = pin(off), pin(tgt), pin(w)
nbytes = off_p.nbytes + tgt_p.nbytes + (w_p.nbytes if w_p is not None else 0)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dg = native.DeviceGraph.from_csr(off_p, tgt_p, w_p)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    lab, log, ms = dg.run(params)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del dg
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):7.1f} ms ({nbytes/(t1-t0)/1e9:5.1f} GB/s)  run+labels {1e3*(t2-t1):6.1f} ms"
          f" (device {ms:5.2f} ms)  destroy {1e3*(t3-t2):5.1f} ms", flush=True)
x = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda")
h = torch.empty(nbytes // 4, dtype=torch.int32).pin_memory()
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    print(f"raw pinned H2D {nbytes/(time.perf_counter()-t0)/1e9:.1f} GB/s")
