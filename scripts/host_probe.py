"""Host-side facts of the GPU box that bound the e2e path: cores, RAM,
host memory bandwidth (torch CPU copy, all threads) and pinned H2D/D2H."""
import json, os, time
import torch

def bw(fn, nbytes, reps=5):
    best = 1e9
    for _ in range(reps):
        t = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return nbytes / best / 1e9

n = 1 << 30
a = torch.empty(n, dtype=torch.uint8).fill_(1)
b = torch.empty(n, dtype=torch.uint8)
info = {"nproc": os.cpu_count(), "torch_threads": torch.get_num_threads(),
        "mem_total_gb": os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9}
info["host_copy_GBps"] = bw(lambda: b.copy_(a), 2 * n)
p = torch.empty(n, dtype=torch.uint8, pin_memory=True).fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
info["h2d_pinned_GBps"] = bw(lambda: d.copy_(p, non_blocking=True), n)
info["d2h_pinned_GBps"] = bw(lambda: p.copy_(d, non_blocking=True), n)
info["h2d_pageable_GBps"] = bw(lambda: d.copy_(a), n, reps=3)
x64 = torch.randint(1, 64, (n // 8,), dtype=torch.int64)
y8 = torch.empty(n // 8, dtype=torch.uint8)
info["host_i64_to_u8_GBps_read"] = bw(lambda: y8.copy_(x64), n)
print(json.dumps(info))
