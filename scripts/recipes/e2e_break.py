import sys, time, numpy as np, torch
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1911_09135_b200 as sg
from paper_1911_09135_b200 import native
g = sg.attach_random_weights(sg.generate_rmat(24, 16, 1), 2)
dev = g.device()
off, tgt, w = dev.download(0, weights=True)
print("dtypes", off.dtype, tgt.dtype, w.dtype, off.flags['C_CONTIGUOUS'], tgt.flags['C_CONTIGUOUS'], w.flags['C_CONTIGUOUS'])
pin = lambda x: torch.from_numpy(x).pin_memory().numpy()
off_p, tgt_p, w_p = pin(off), pin(tgt), pin(w)
print("bytes", off_p.nbytes + tgt_p.nbytes + w_p.nbytes)
params = native.RunParams() if hasattr(native, "RunParams") else None
import bench
_, params = bench.run_params(sg, "sssp", "alb", None, dev.info()[0])
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dg = native.DeviceGraph.from_csr(off_p, tgt_p, w_p)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    lab, log, ms = dg.run(params)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    del dg
    print(f"create {1e3*(t1-t0):.1f} ms  run+labels {1e3*(t2-t1):.1f} ms (device {ms:.2f})")
# raw pinned copy bandwidth
x = torch.empty(w_p.nbytes, dtype=torch.uint8, device="cuda")
src = torch.from_numpy(w_p.view(np.uint8))
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); x.copy_(src, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"raw H2D {w_p.nbytes/1e9:.2f} GB in {1e3*(t1-t0):.1f} ms = {w_p.nbytes/(t1-t0)/1e9:.1f} GB/s")
