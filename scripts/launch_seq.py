"""Print the kernel sequence (per-launch us) of the last SSSP run in an ncu
launch list: python scripts/launch_seq.py gpurun_out/TAG_launches.csv [marker] [n]"""
import csv
import sys

path = sys.argv[1]
marker = sys.argv[2] if len(sys.argv) > 2 else "k_bm_twc<BmMin<2>"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 52
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
seq = [(r[ki].split("(")[0].replace("void ", "").replace("sg::", "").replace("<unnamed>::", ""),
        float(r[vi].replace(",", ""))) for r in rows[hdr + 1:] if len(r) > vi]
idx = [i for i, (k, v) in enumerate(seq) if k.startswith(marker) and v > 100000]
s = idx[-3] - 12 if len(idx) >= 3 else 0
tot = 0.0
for k, v in seq[s:s + n]:
    print(f"{v / 1000:8.1f} us  {k[:64]}")
    tot += v
print(f"total {tot / 1000:.1f} us")
