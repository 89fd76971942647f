"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes) per kernel."""
import csv
import re
import sys
from collections import OrderedDict, defaultdict

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].strip('"').isdigit()]
launch = OrderedDict()
for r in rows:
    lid = int(r[0])
    name = re.sub(r"\(.*", "", r[4]).replace("void ", "").replace("unnamed>::", "")
    launch.setdefault(lid, {"name": name, "grid": r[8], "block": r[7]})
    launch[lid][r[-3]] = float(r[-1].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
total = 0.0
for lid, d in launch.items():
    t = d.get("gpu__time_duration.sum", 0.0)
    a = agg[d["name"]]
    a[0] += 1
    a[1] += t
    a[2] += d.get("dram__bytes_read.sum", 0.0)
    a[3] += d.get("dram__bytes_write.sum", 0.0)
    total += t
print(f"{'kernel':40s} {'n':>3s} {'avg_us':>9s} {'share':>6s} {'rd_MB':>9s} {'wr_MB':>9s} {'GB/s':>8s}")
for name, (n, t, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    gbs = (rd + wr) / t if t else 0.0  # bytes/ns = GB/s
    print(f"{name:40s} {n:3d} {t / n / 1e3:9.1f} {100 * t / total:5.1f}% {rd / n / 1e6:9.1f} {wr / n / 1e6:9.1f} {gbs:8.0f}")
