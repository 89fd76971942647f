"""profiles/ncu_traffic.json from an ncu launch list: DRAM bytes per pixel for each kernel."""
import csv
import json
import re
import sys
from collections import defaultdict

path, npx_total = sys.argv[1], float(sys.argv[2])
rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].strip('"').isdigit()]
per = defaultdict(lambda: defaultdict(float))
launch_name = {}
for r in rows:
    lid = int(r[0])
    name = re.sub(r"<.*", "", re.sub(r"\(.*", "", r[4]).replace("void ", "").replace("unnamed>::", "")).strip()
    launch_name[lid] = name
    per[lid][r[-3]] = float(r[-1].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for lid, m in per.items():
    a = agg[launch_name[lid]]
    a[0] += 1
    a[1] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a[2] += m.get("gpu__time_duration.sum", 0.0)
out = {"source": path, "pixels_per_launch": npx_total,
       "kernels": {k: {"launches": n, "dram_bytes_per_px": round(b / n / npx_total, 4),
                       "avg_us": round(t / n / 1000.0, 2)} for k, (n, b, t) in agg.items()}}
print(json.dumps(out, indent=1))
