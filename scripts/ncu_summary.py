"""Summarise ncu outputs (launch list CSV + --set full report) into profiles/.

usage: python scripts/ncu_summary.py TAG --workload sssp/rmat24
reads  gpurun_out/TAG_launches.csv, gpurun_out/TAG_prof.ncu-rep
writes profiles/TAG_ncu.json (+ updates profiles/ncu_summary.json, which
bench.py reads for roofline.traffic)
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
]


def short(name):
    n = name.replace("(int)", "").replace("(bool)", "").split("(")[0]
    for junk in ("void ", "sg::", "<unnamed>::", "(anonymous namespace)::"):
        n = n.replace(junk, "")
    return n


def launches(tag):
    p = ROOT / "gpurun_out" / f"{tag}_launches.csv"
    if not p.exists():
        return None
    rows = list(csv.reader(open(p)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        a = agg.setdefault(short(r[ki]), [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", "")) / 1e3
    tot = sum(a[1] for a in agg.values())
    return {k: {"launches": a[0], "us": round(a[1], 1), "share": round(a[1] / tot, 4)}
            for k, a in sorted(agg.items(), key=lambda x: -x[1][1])}


def full(tag):
    p = ROOT / "gpurun_out" / f"{tag}_prof.ncu-rep"
    if not p.exists():
        return None
    out = subprocess.run(["ncu", "-i", str(p), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for m in METRICS:
            if m in h:
                v = r[h.index(m)].replace(",", "")
                try:
                    d[m] = float(v)
                except ValueError:
                    d[m] = v
        res.append(d)
    return res


def main():
    tag = sys.argv[1]
    wl = sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv else "sssp/rmat24"
    summary = {"tag": tag, "launch_list": launches(tag), "full": full(tag)}
    per = collections.defaultdict(list)
    for d in summary["full"] or []:
        unit_scale = 1.0  # ncu raw csv reports dram bytes in the unit of row 1 (we read Mbyte/Gbyte)
        per[d["kernel"].split("<")[0]].append(d)
    summary["dram_bytes_per_launch"] = {}
    units = None
    rep = ROOT / "gpurun_out" / f"{tag}_prof.ncu-rep"
    if rep.exists():
        out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        units = dict(zip(rows[0], rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for k, lst in per.items():
        b = [d.get("dram__bytes_read.sum", 0) * scale[units["dram__bytes_read.sum"]]
             + d.get("dram__bytes_write.sum", 0) * scale[units["dram__bytes_write.sum"]] for d in lst]
        t = [d.get("gpu__time_duration.sum", 0) for d in lst]
        summary["dram_bytes_per_launch"][f"{k}|{wl}"] = sum(b) / len(b)
        summary.setdefault("captured_launches", {})[k] = {"n": len(lst), "dram_bytes": b,
                                                          "time": t,
                                                          "time_unit": units["gpu__time_duration.sum"]}
    outp = ROOT / "profiles" / f"{tag}_ncu.json"
    outp.write_text(json.dumps(summary, indent=1) + "\n")
    agg = ROOT / "profiles" / "ncu_summary.json"
    prev = json.loads(agg.read_text()) if agg.exists() else {}
    prev.setdefault("dram_bytes_per_launch", {}).update(summary["dram_bytes_per_launch"])
    prev.setdefault("sources", {}).update({k: f"profiles/{tag}_ncu.json"
                                           for k in summary["dram_bytes_per_launch"]})
    prev["note"] = ("dram bytes per launch (ncu --set full) keyed 'kernel|workload'; bench.py "
                    "reports traffic only for the workload a kernel was captured on")
    agg.write_text(json.dumps(prev, indent=1) + "\n")
    print(json.dumps({k: v for k, v in summary.items() if k != "full"}, indent=1)[:3000])


if __name__ == "__main__":
    main()
