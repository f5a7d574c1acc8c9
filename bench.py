"""Benchmark: ALB SSSP on RMAT scale-24 (integer weights), GTEPS on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W``; N>1 is
launched under torchrun (one rank per GPU).  Rank 0 prints ONE JSON line.

Workload (BASELINE.json configs[1]): SSSP from source 0 on
generate_rmat(24, 16, seed=1, (0.57,0.19,0.19,0.05)) with
attach_random_weights(seed=2) integers in [1, 64]; scheduler alb (cyclic,
threshold = KernelConfig().total_threads = 21,504).  One step = one complete
BSP run (all rounds to convergence) of the device engine.

* value  : GTEPS = edges_processed (the reference's report totals,
           engine.py:293) x K / sum of per-step device times; inputs resident
           in HBM; L2 flushed (512 MB write) before every step; each step timed
           with CUDA events on the engine's stream (sg_run, SG_FLAG_TIMING);
           max over ranks.
* e2e    : the same metric through the C ABI with HOST buffers: per step
           sg_graph_create from pinned CSR/weights (H2D) + sg_run + labels /
           round log D2H, wall clock with device sync.
* layout : the resident graph is re-run, so from the second warm-up run on the
           engine uses its hot-vertex relabeled store (labels and
           round logs in the reference's numbering); e2e builds a fresh graph
           every step, which is run once in its original numbering.
* roofline: dominant kernel of a profiled run (sg_run_profiled: CUDA events
           around every kernel) — algorithmic bytes / its time,
           against MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline: the C oracle (oracle/sg_oracle.c, a restatement of the
           reference path) on this host, 1 thread, full workload.
* labels : every workload's float64 labels are hashed (sha256, the
           reference's numbering) and compared with tests/golden/
           scale_golden.json (the C oracle pinned to the reference) together
           with the round count -- pr included (bit-exact sums, sg_prx.cuh).
* configs: BASELINE.json configs[2..4] at their own scales on this GPU --
           C3 cc rmat25, C4 pr rmat25 skewed and uniform, C5 bfs / kcore
           rmat27 -- each with its label check, dominant-kernel roofline and
           ALB / TWC-only ratio.
* ablation_heavy_skew: ALB vs TWC-only on rmat24 with the reference's
           probabilities knob at (0.8, 0.1, 0.05, 0.05) (graph.py:274,
           cli.py:113-114), every app, labels checked.
``--impl reference`` times that CPU path alone with all host threads.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GTEPS for BFS/SSSP/CC/PR on RMAT power-law graphs at 1/2/4/8 B200"
SKEWED = (0.57, 0.19, 0.19, 0.05)
HEAVY = (0.8, 0.1, 0.05, 0.05)   # SURVEY §7.6 heavier skew (the reference's probabilities knob)
DEFAULT_THRESHOLD = 84 * 256  # KernelConfig().total_threads (simt.py:20-22)

# algorithmic bytes (SURVEY §8d canonical widths)
EDGE_BYTES = {"bfs": 8, "cc": 8, "sssp": 12, "kcore": 8, "pr": 12}
VERTEX_BYTES = 24   # frontier id 4 + offsets 16 + snapshot label 4
UPDATE_BYTES = 8    # label write 4 + enqueue 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--app", default="sssp", choices=["bfs", "sssp", "cc", "pr", "kcore"])
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--uniform", action="store_true", help="uniform RMAT probabilities")
    ap.add_argument("--probs", default=None,
                    help="RMAT probabilities a,b,c,d (the reference's --rmat-probs), e.g. 0.8,0.1,0.05,0.05")
    ap.add_argument("--sched", default="alb", choices=["alb", "twc"])
    ap.add_argument("--threshold", type=int, default=DEFAULT_THRESHOLD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--extra", default="bfs,cc,pr,kcore",
                    help="comma list of extra apps reported on the same rmat graph ('' = none)")
    ap.add_argument("--no-ablation", action="store_true",
                    help="skip the ALB vs TWC-only (classic / batched CTA bin) ablation")
    ap.add_argument("--pr-block", type=int, default=0,
                    help="pr source-block size in vertices (0 = automatic, -1 = never tile)")
    ap.add_argument("--cta-bin", default="batched", choices=["batched", "classic"],
                    help="TWC CTA bin: edge-balanced batches (default) or one vertex per CTA")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the BASELINE configs C3-C5 at their own scales")
    ap.add_argument("--no-heavy", action="store_true",
                    help="skip the heavy-skew ALB vs TWC-only ablation")
    ap.add_argument("--peer", action="store_true",
                    help="N=1: run the multi-GPU code path (partition + NVLink peer team of one "
                         "rank, device barrier, label gather) instead of sg_run")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


class Clocks:
    """SM clock + throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line): NVML polled every 2 ms from a thread
    (the timed region is only tens of ms), nvidia-smi as the fallback."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.sm, self.mx, self.reasons = [], 0.0, set()
        self.stop = threading.Event()
        self.nvml = None

    def _sample_nvml(self):
        import pynvml as N
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        h = self.nvml
        self.mx = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
        while True:
            self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
            r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.reasons.update(n for n, bit in bits.items() if r & bit)
            if self.stop.wait(0.002):
                break

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout
                parts = [x.strip() for x in out.split(",")]
                self.sm.append(float(parts[0]))
                self.mx = max(self.mx, float(parts[1]))
                self.reasons.update(n for n, v in zip(self.NAMES, parts[2:6])
                                    if v.lower().startswith("active"))
            except (OSError, ValueError, IndexError, subprocess.TimeoutExpired):
                return

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.nvml = N.nvmlDeviceGetHandleByIndex(self.index)
            target = self._sample_nvml
        except Exception:  # noqa: BLE001 - no NVML: nvidia-smi polling
            target = self._sample_smi
        self.t = threading.Thread(target=target, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        sm = self.sm
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.mx or None,
                "reasons": sorted(self.reasons), "samples": len(sm),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def algorithmic_bytes(app, log, dense0=False):
    """Per-kernel algorithmic bytes from the round log.
    dense0: cc's round 0 ran as the streaming pull k_cc_dense (col 4 B / edge,
    offsets 16 B / row, label + bitmap 8 B / changed vertex)."""
    if app == "cc" and dense0 and len(log):
        rest = algorithmic_bytes(app, log[1:])
        m0, n0, u0 = (int(log["active_edges"][0]), int(log["frontier_size"][0]),
                      int(log["updated"][0]))
        rest["cc_dense"] = 4 * m0 + 16 * n0 + UPDATE_BYTES * u0
        rest["compact"] = rest.get("compact", 0) + UPDATE_BYTES * u0
        return rest
    eb = EDGE_BYTES[app]
    n = log["frontier_size"].astype(np.int64)
    m = log["active_edges"].astype(np.int64)
    mh = log["huge_edges"].astype(np.int64)
    ml = log["large_edges"].astype(np.int64)
    u = log["updated"].astype(np.int64)
    if app == "pr":  # one exact-order pull kernel per round (sg_prx.cuh)
        nv = int(n[0]) if len(n) else 0
        return {"pr_pull": int((eb * m).sum() + 40 * nv * len(n))}
    if app == "kcore":
        return {"pull_twc": int((eb * (m - mh - ml) + VERTEX_BYTES * n).sum()),
                "pull_large": int((eb * ml).sum()), "pull_lb": int((eb * mh).sum())}
    return {"push_twc": int((eb * (m - mh - ml) + VERTEX_BYTES * n).sum()),
            "push_large": int((eb * ml).sum()), "push_lb": int((eb * mh).sum()),
            "compact": int((UPDATE_BYTES * u).sum())}


def kernel_edges(log):
    """Edges (operator applications) per traversal kernel from the round log."""
    m = log["active_edges"].astype(np.int64)
    mh = log["huge_edges"].astype(np.int64)
    ml = log["large_edges"].astype(np.int64)
    return {"twc": int((m - mh - ml).sum()), "large": int(ml.sum()), "lb": int(mh.sum()),
            "pull": int(m.sum())}


# profiled-run kernel names -> the CUDA kernels ncu lists
NCU_NAME = {"push_twc": "k_bm_twc", "push_large": "k_bm_large_pipe", "push_lb": "k_bm_lb",
            "compact": "k_bm_compact", "pull_twc": "k_pull_twc", "pull_large": "k_pull_large",
            "pull_lb": "k_pull_lb", "pr_pull": "k_prx", "cc_dense": "k_cc_dense"}
# random 4-byte gathers per second the chip sustains (scripts/micro/gather.cu on
# B200: 272-275 G/s, one L1TEX wavefront per scattered lane)
GATHER_CEILING = 272e9


def total_algorithmic_bytes(app, log, nv):
    b = algorithmic_bytes(app, log)
    return sum(b.values())


def ncu_traffic(kernel, workload):
    """dram bytes per launch of `kernel` on `workload` from the committed ncu
    summaries (profiles/ncu_summary.json, keyed "kernel|workload"); null when
    that kernel was not captured on that workload."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        key = f"{kernel}|{workload}"
        b = d.get("dram_bytes_per_launch", {}).get(key)
        if b is None:
            return None
        return {"dram_bytes_per_launch": b,
                "launches_captured": d.get("launches_captured", {}).get(key),
                "source": d.get("sources", {}).get(key)}
    except (ValueError, OSError):
        return None


def workload_name(app, scale, probs):
    kind = "uniform" if tuple(probs) == (0.25,) * 4 else "heavy" if tuple(probs) == HEAVY else "rmat"
    return f"{app}/{kind}{scale}"


_GOLDEN = None


def scale_golden():
    global _GOLDEN
    if _GOLDEN is None:
        p = ROOT / "tests" / "golden" / "scale_golden.json"
        _GOLDEN = json.loads(p.read_text()) if p.exists() else {}
    return _GOLDEN


def label_check(key, labels, log):
    """sha256 of the float64 labels and the round count vs the committed golden."""
    import hashlib
    info = scale_golden().get(key)
    if info is None:
        return {"golden": None}
    sha = hashlib.sha256(np.ascontiguousarray(labels, dtype=np.float64).tobytes()).hexdigest()
    return {"labels_match": sha == info["labels_sha256"], "rounds_match": len(log) == info["rounds"],
            "rounds": len(log), "golden_rounds": info["rounds"], "golden": "tests/golden/scale_golden.json:" + key}


def roofline_of(app, kernels, plog, step_ms, workload):
    """Dominant kernel of a profiled run vs the measured HBM peak."""
    ab = algorithmic_bytes(app, plog, dense0="cc_dense" in kernels)
    timed = {k: v for k, v in kernels.items() if k in ab}
    if not timed:
        return None
    dom = max(timed, key=lambda k: timed[k][1])
    peak, peak_kind = peaks()
    n_l, ms_l = kernels[dom]
    achieved = ab[dom] / (ms_l / 1e3) / 1e9
    name = NCU_NAME.get(dom, dom)
    tr = ncu_traffic(name, workload)
    ke = (int(plog["active_edges"][0]) if dom == "cc_dense" else
          kernel_edges(plog).get("pull" if dom == "pr_pull" else dom.split("_")[-1], 0))
    return {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_source": peak_kind,
            "traffic": (tr or {}).get("dram_bytes_per_launch"),
            "traffic_launches_captured": (tr or {}).get("launches_captured"),
            "algorithmic_bytes_per_launch": ab[dom] / max(n_l, 1),
            "avg_launch_ms": ms_l / max(n_l, 1), "launches": n_l,
            "share_of_step": ms_l / sum(v[1] for v in kernels.values()),
            "loop_bytes_per_s_GBps": sum(ab.values()) / (step_ms / 1e3) / 1e9,
            "loop_frac": sum(ab.values()) / (step_ms / 1e3) / 1e9 / peak,
            "gather_rate": {"unit": "G label accesses/s", "achieved": ke / (ms_l / 1e3) / 1e9,
                            "uncached_microbench": GATHER_CEILING / 1e9,
                            "ratio_to_uncached": ke / (ms_l / 1e3) / GATHER_CEILING,
                            "note": "scattered 4-byte gathers that miss L1 (scripts/micro/"
                                    "gather.cu, B200): a reference rate, not a bound -- "
                                    "kernels whose hot labels hit L1 exceed it"}}


def make_graph_device(sg, app, scale, uniform, probs=None):
    probs = probs or ((0.25,) * 4 if uniform else SKEWED)
    g = sg.generate_rmat(scale, 16, 1, probs)
    return (sg.attach_random_weights(g, 2) if app == "sssp" else g), g


def run_params(sg, app, sched_kind, threshold, nv, classic=False):
    sched = sg.Scheduler(sched_kind, threshold=threshold if sched_kind == "alb" else None)
    p = sg.engine.device_params(sg.apps.make_app(app), sched, sg.KernelConfig(), 1, 10 * nv + 256)
    if classic:
        p.flags |= 4  # SG_FLAG_TWC_CLASSIC
    return sched, p


def device_steps(torch, dev, params, steps, warmup, flush, keep=False):
    """W untimed + K timed BSP runs; per-run CUDA-event time of sg_run, L2 flushed before each."""
    for _ in range(max(1, warmup)):
        labels, log, ms = dev.run(params)
    out = []
    for i in range(steps):
        flush.fill_(i & 0xFF)
        torch.cuda.synchronize()
        labels, log, ms = dev.run(params)
        out.append(ms)
    edges = int(log["active_edges"].sum())
    r = {"gteps": edges * len(out) / (sum(out) / 1e3) / 1e9,
         "ms_per_step": sum(out) / len(out), "rounds": len(log), "edges_processed": edges}
    if keep:
        r["_labels"], r["_log"] = labels, log
    return r


def config_entry(sg, torch, app, scale, probs, flush, threshold, steps, ablate=True,
                 classic=True):
    """One workload at its own scale: ALB runs (the graph stays resident, so
    from the second run on it uses the relabeled store), labels vs the golden,
    the dominant kernel's roofline, ALB / TWC-only.  The graph is dropped after."""
    from paper_1911_09135_b200 import native
    t0 = time.perf_counter()
    g, _ = make_graph_device(sg, app, scale, False, probs)
    dev = g.device()
    nv, ne, _ = dev.info()
    gen_s = time.perf_counter() - t0
    wl = workload_name(app, scale, probs)
    first = dev.run(run_params(sg, app, "alb", threshold, nv)[1])
    r = device_steps(torch, dev, run_params(sg, app, "alb", threshold, nv)[1], steps, 1, flush,
                     keep=True)
    chk = label_check(wl, r.pop("_labels"), r.pop("_log"))
    _, plog, pms, kernels = dev.run(run_params(sg, app, "alb", threshold, nv)[1], profile=True)
    out = {"workload": wl, "num_vertices": nv, "num_edges": ne, **r, **chk,
           "value_first_run": r["edges_processed"] / (first[2] / 1e3) / 1e9,
           "build_ms": {k: round(v, 1) for k, v in dev.build_ms().items()},
           "generate_s": round(gen_s, 2),
           "roofline": roofline_of(app, kernels, plog, r["ms_per_step"], wl)}
    if ablate:
        tw = device_steps(torch, dev, run_params(sg, app, "twc", None, nv)[1], steps, 1, flush)
        out["twc_gteps"] = tw["gteps"]
        out["alb_over_twc"] = r["gteps"] / tw["gteps"]
        if classic and app != "pr":
            twc_c = device_steps(torch, dev, run_params(sg, app, "twc", None, nv, True)[1], steps,
                                 1, flush)["gteps"]
            alb_c = device_steps(torch, dev, run_params(sg, app, "alb", threshold, nv, True)[1],
                                 steps, 1, flush)["gteps"]
            out["classic_cta_bin"] = {"alb_gteps": alb_c, "twc_gteps": twc_c,
                                      "alb_over_twc": alb_c / twc_c, "alb_over_twc_classic": r["gteps"] / twc_c}
    del dev, g
    import gc
    gc.collect()
    native.load().sg_release_cached()
    return {k: (round(v, 4) if isinstance(v, float) else v) for k, v in out.items()}


def cpu_oracle_run(app, off, tgt, w, threads):
    from oracle import oracle_c as C
    args = C.prepare(off, tgt, w, app)
    t0 = time.perf_counter()
    lab, log, st = C.run(app, *args, threads=threads)
    dt = time.perf_counter() - t0
    return lab, log, dt


def run_reference(a):
    """--impl reference: the reference path (C restatement) on host cores."""
    rank, _, world = dist_env()
    if world > 1 and rank != 0:
        return
    from oracle import oracle_c as C
    from oracle import oracle_np as O
    threads = os.cpu_count() or 1
    probs = (0.25,) * 4 if a.uniform else SKEWED
    s, d = C.rmat_pairs(a.scale, 16, 1, probs, threads=threads)
    w = O.random_weights(len(s), 2) if a.app == "sssp" else None
    off, tgt, _ = C.csr_from_pairs(s, d, 1 << a.scale)
    del s, d
    args = C.prepare(off, tgt, w, a.app)
    times, edges = [], 0
    for i in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        lab, log, st = C.run(a.app, *args, threads=threads)
        dt = time.perf_counter() - t0
        if i >= a.warmup:
            times.append(dt)
            edges = int(log[:, 1].sum())
    total = sum(times)
    value = edges * len(times) / total / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"{a.app} rmat{a.scale} ef16 seed1" + (" uniform" if a.uniform else "")
                   + (" weights[1,64] seed2" if a.app == "sssp" else "") + " source0",
                   "edges_processed": edges, "scheduler": "n/a (CPU restatement)"},
        "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": threads, "kind": "port",
                         "sample": f"full {a.app} run on rmat{a.scale}, oracle/sg_oracle.c "
                                   f"(OpenMP, {threads} threads)"},
        "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.peer:  # the multi-GPU code path alone: no single-device sections
        a.no_cpu_baseline = a.no_ablation = a.no_configs = a.no_heavy = True
        a.extra = ""
    if a.impl == "reference":
        return run_reference(a)
    rank, local_rank, world = dist_env()
    import torch
    import paper_1911_09135_b200 as sg
    from paper_1911_09135_b200 import dist as sgdist
    from paper_1911_09135_b200 import native
    device = sgdist.init_device() if world > 1 else local_rank
    torch.cuda.set_device(device)
    if world > 1:  # plumbing only (IPC handle exchange, max over ranks); gloo when
        import torch.distributed as dist  # ranks share a GPU (NCCL refuses duplicate GPUs)
        if native.device_count() >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group("gloo")

    probs = tuple(float(x) for x in a.probs.split(",")) if a.probs else None
    g, g_base = make_graph_device(sg, a.app, a.scale, a.uniform, probs)
    dev = g.device()
    nv, ne, _ = dev.info()
    sched, params = run_params(sg, a.app, a.sched, a.threshold, nv, a.cta_bin == "classic")
    params.reserved = a.pr_block if a.pr_block > 0 else (1 << 31) - 1 if a.pr_block < 0 else 0
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    team = part = None
    if world > 1 or a.peer:
        # edge cut over NVLink peer memory: this rank keeps only its rows (the
        # full graph is generated, sliced and dropped), the label exchange is
        # done by the round's kernels in the peers' HBM (sg_peer.cu)
        params.devices = world
        part = sgdist.partition(g if a.app == "sssp" else g_base, a.app, rank, world)
        host_csr = None if a.no_e2e else dev.download(0, weights=(a.app == "sssp"))
        del g, g_base, dev
        native.release_cached()
        if world > 1:
            team = sgdist.make_team(torch.distributed, nv)
        else:
            team = native.Team(0, 1, nv)
        dev = part.device()

    def step(d):
        if team is not None:
            return team.run(d, params)
        return d.run(params)

    warm_ms = []
    for _ in range(max(1, a.warmup)):
        labels, log, ms = step(dev)
        warm_ms.append(ms)
    edges = int(log["active_edges"].sum())
    rounds = len(log)
    workload = workload_name(a.app, a.scale, probs or ((0.25,) * 4 if a.uniform else SKEWED))

    # ---------------- timed region (device-resident inputs) ----------------
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = native.kernel_launches()
    step_ms = []
    t_wall = time.perf_counter()
    with Clocks(local_rank) as clk:
        for i in range(a.steps):
            flush.fill_(i & 0xFF)  # evict L2 (> 126 MB) between steps
            torch.cuda.synchronize()
            labels, log2, ms = step(dev)
            step_ms.append(ms)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall
    launches = native.kernel_launches() - launches0
    total_ms = sum(step_ms)
    if world > 1:
        total_ms = sgdist.max_over_ranks(torch.distributed, total_ms)
    # whole-job throughput: the (fixed) graph's processed edges per second
    value = edges * a.steps / (total_ms / 1e3) / 1e9
    check = label_check(workload, labels, log2) if rank == 0 else None

    # ---------------- e2e through the C ABI with host buffers ----------------
    e2e = None
    if not a.no_e2e:
        off, tgt, w = host_csr if team is not None else dev.download(0, weights=(a.app == "sssp"))
        pin = lambda x: torch.from_numpy(x).pin_memory().numpy() if x is not None else None
        off_p, tgt_p, w_p = pin(off), pin(tgt), pin(w)
        # sg_graph_create packs weights in [0, 255] / [0, 65535] into 1 / 2 bytes
        # on the host before the copy (sg_engine.cu upload_weights)
        wbytes = 0
        if w_p is not None and len(w_p):
            lo_w, hi_w = int(w_p.min()), int(w_p.max())
            wbytes = len(w_p) * (1 if lo_w >= 0 and hi_w <= 255 else
                                 2 if lo_w >= 0 and hi_w <= 65535 else 8)
        h2d = off_p.nbytes + tgt_p.nbytes + wbytes
        d2h = 8 * nv + native.ROUND_DTYPE.itemsize * rounds
        def upload():
            dg = native.DeviceGraph.from_csr(off_p, tgt_p, w_p)
            if team is None:
                return dg
            kind = sgdist.PART_KIND[a.app]
            return native.DevicePartition.of(dg, kind, world, rank)

        # warm-up with the timed loop's own pattern: the previous step's labels
        # (a pinned block of the library's host pool) are alive while the next
        # run fills a new one, so the pool settles at two blocks before timing
        lab_e = None
        for _ in range(3):
            dg = upload()
            lab_e, log_e, _ = step(dg)
            del dg
        torch.cuda.synchronize()
        e2e_s, up_s = [], []
        for _ in range(max(1, a.steps)):
            t0 = time.perf_counter()
            dg = upload()
            up_s.append(time.perf_counter() - t0)
            lab_e, log_e, _ = step(dg)
            torch.cuda.synchronize()
            e2e_s.append(time.perf_counter() - t0)
            del dg
        e2e_tot = sum(e2e_s)
        if world > 1:
            e2e_tot = sgdist.max_over_ranks(torch.distributed, e2e_tot)
        e2e = {"value": edges * len(e2e_s) / e2e_tot / 1e9, "unit": "GTEPS",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * e2e_tot / len(e2e_s), "steps": len(e2e_s),
               "upload_ms_median": 1e3 * statistics.median(up_s),
               "step_ms": [round(1e3 * x, 1) for x in e2e_s],
               "note": "per step: sg_graph_create from pinned host CSR (+ int64 weights, packed "
                       "to their byte width on the host while the topology is in flight), sg_run "
                       "(original numbering: a fresh graph's first run), labels + round log D2H"
                       if team is None else
                       "per step and rank: sg_graph_create of the full CSR (+ int64 weights) "
                       "from pinned host memory, sg_graph_partition (this rank's rows), "
                       "sg_team_run, labels + round log D2H; max over ranks"}
        assert np.array_equal(lab_e, labels)

    # ---------------- roofline from a profiled run ----------------
    roofline, kernels = None, {}
    if team is None:
        _, plog, pms, kernels = dev.run(params, profile=True)
        roofline = roofline_of(a.app, kernels, plog, statistics.median(step_ms), workload)

    # ---------------- CPU baseline (rank 0, N=1 only) ----------------
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        off, tgt, w = dev.download(0, weights=(a.app == "sssp"))
        lab_c, log_c, dt = cpu_oracle_run(a.app, off, tgt, w, threads=1)
        e_c = int(log_c[:, 1].sum())
        cpu = {"value": e_c / dt / 1e9, "unit": "GTEPS", "cores": 1, "kind": "port",
               "sample": f"full {a.app} run on the same rmat{a.scale} graph, "
                         f"oracle/sg_oracle.c single thread ({dt:.1f} s)",
               "labels_match": bool(np.array_equal(lab_c, labels))}

    # ------------- other apps + ALB vs TWC-only ablation (rank 0, N=1) -------------
    extra, ablation = {}, {}
    if rank == 0 and world == 1:
        steps_x = max(2, min(a.steps, 3))
        apps = [x for x in a.extra.split(",") if x]
        for app in apps:
            d = g.device() if app == "sssp" else g_base.device()
            r = device_steps(torch, d, run_params(sg, app, "alb", a.threshold, nv)[1], steps_x, 1,
                             flush, keep=True)
            wl = workload_name(app, a.scale, (0.25,) * 4 if a.uniform else SKEWED)
            r.update(label_check(wl, r.pop("_labels"), r.pop("_log")))
            _, pl, _, ks = d.run(run_params(sg, app, "alb", a.threshold, nv)[1], profile=True)
            rf = roofline_of(app, ks, pl, r["ms_per_step"], wl)
            if rf:
                r["roofline"] = {k: rf[k] for k in ("kernel", "achieved", "frac", "traffic",
                                                    "share_of_step", "loop_frac")}
            extra[app] = r
        if not a.no_ablation:
            for app in sorted(set([a.app] + apps)):
                d = g.device() if app == "sssp" else g_base.device()
                alb = extra[app]["gteps"] if app in extra else value
                tw_b = device_steps(torch, d, run_params(sg, app, "twc", None, nv)[1], steps_x, 1,
                                    flush)["gteps"]
                ablation[app] = {"alb_gteps": alb, "twc_gteps": tw_b, "alb_over_twc": alb / tw_b}
                if app != "pr":  # the exact pr kernel has one CTA-bin form (sg_prx.cuh)
                    tw_c = device_steps(torch, d, run_params(sg, app, "twc", None, nv, True)[1],
                                        steps_x, 1, flush)["gteps"]
                    alb_c = device_steps(torch, d,
                                         run_params(sg, app, "alb", a.threshold, nv, True)[1],
                                         steps_x, 1, flush)["gteps"]
                    ablation[app]["classic_cta_bin"] = {"alb_gteps": alb_c, "twc_gteps": tw_c,
                                                        "alb_over_twc": alb_c / tw_c}

    # hardware load balance (paper Fig. 1 / 7 analogue): per-round edges per SM
    # from sg_run_cta_counts, worst round's max/mean and CV
    if rank == 0 and world == 1 and not a.no_ablation:
        def cta_load(kind, classic):
            _, lg, _, cta = dev.run_cta_counts(run_params(sg, a.app, kind, a.threshold, nv,
                                                          classic)[1])
            worst_mm, worst_cv, heavy = 0.0, 0.0, None
            for r in range(len(cta)):
                row = cta[r].astype(np.float64)
                if row.sum() < 1e6:  # rounds with real work only
                    continue
                mm, cv = row.max() / row.mean(), row.std() / row.mean()
                if mm > worst_mm:
                    worst_mm, worst_cv, heavy = mm, cv, r
            return {"worst_round": heavy, "max_over_mean": round(worst_mm, 3),
                    "cv": round(worst_cv, 3), "sms": int(cta.shape[1]) if len(cta) else 0}
        ablation.setdefault(a.app, {})["cta_load"] = {
            "alb": cta_load("alb", False), "twc": cta_load("twc", False),
            "alb_classic_cta_bin": cta_load("alb", True), "twc_classic": cta_load("twc", True)}

    # every scheduler of the reference on the headline workload (paper Table 3)
    schedulers = {}
    if rank == 0 and world == 1 and not a.no_ablation:
        for kind in ("vertex", "edge", "lb", "twc", "alb"):
            schedulers[kind] = round(device_steps(
                torch, dev, run_params(sg, a.app, kind, a.threshold, nv)[1],
                max(2, min(a.steps, 3)), 1, flush)["gteps"], 2)
    build_ms = {k: round(v, 1) for k, v in dev.build_ms().items()}
    value_first_run = edges / (warm_ms[0] / 1e3) / 1e9

    # --------- the graphs of the other BASELINE configs / the skew ablation ---------
    heavy, configs = {}, {}
    if rank == 0 and world == 1 and (not a.no_heavy or not a.no_configs):
        del dev, g, g_base
        import gc
        gc.collect()
        native.load().sg_release_cached()
        steps_c = 2
        if not a.no_heavy:  # the paper's >= 1.5x claim needs real skew
            for app in ("bfs", "sssp", "cc", "pr", "kcore"):
                heavy[app] = config_entry(sg, torch, app, 24, HEAVY, flush, a.threshold, steps_c)
        if not a.no_configs:
            for key, (app, scale, probs) in (("C3_cc_rmat25", ("cc", 25, SKEWED)),
                                             ("C4_pr_rmat25", ("pr", 25, SKEWED)),
                                             ("C4_pr_uniform25", ("pr", 25, (0.25,) * 4)),
                                             ("C5_bfs_rmat27", ("bfs", 27, SKEWED)),
                                             ("C5_kcore_rmat27", ("kcore", 27, SKEWED))):
                configs[key] = config_entry(sg, torch, app, scale, probs, flush, a.threshold,
                                            steps_c, classic=False)

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            team.close()
            torch.distributed.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "u32" if a.app in ("bfs", "sssp", "cc") else ("f64" if a.app == "pr" else "u32"),
        "data": "synthetic (device RMAT, bit-identical to the reference's numpy generator)",
        "config": {"workload": f"{a.app} rmat{a.scale} ef16 seed1"
                               + (" uniform" if a.uniform else "")
                               + (" weights[1,64] seed2" if a.app == "sssp" else "")
                               + " source0",
                   "scheduler": sched.describe(), "threshold": a.threshold,
                   "num_vertices": nv, "num_edges": ne, "edges_processed": edges,
                   "rounds": rounds,
                   "parallelism": f"edge-cut x{world}: per-rank partitions, label exchange by "
                                  "the round's kernels over NVLink peer memory, device "
                                  "barrier + quiescence (sg_peer.cu)" if team is not None
                   else "single",
                   "l2": "flushed (512 MB write) before every step",
                   "timing": "sum of per-step CUDA-event durations of sg_run (one graph launch "
                             "per BSP run, float64 labels in the reference's numbering included), "
                             "max over ranks",
                   "wall_s_timed_region": wall},
        "labels": check,
        "value_first_run": value_first_run,
        "build_ms": build_ms,
        "e2e": e2e,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "kernel_ms": {k: {"launches": v[0], "ms": v[1]} for k, v in kernels.items()},
        "apps": {k: {kk: (round(vv, 3) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                 for k, v in extra.items()},
        "ablation_alb_vs_twc": ablation,
        "ablation_heavy_skew": heavy,
        "configs": configs,
        "schedulers_gteps": schedulers,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        team.close()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
