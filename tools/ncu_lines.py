"""Per-source-line totals (instructions executed, stall samples) of one kernel in an ncu report.

usage: python tools/ncu_lines.py REPORT KERNEL_REGEX [TOP]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = None
files = {}
cur_file = None
stats = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    line, src = r[0], r[1]
    if not line.isdigit():
        continue
    try:
        inst = float(r[hdr.index("Instructions Executed")] or 0)
        samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    key = (cur_file.rsplit("/", 1)[-1], int(line), src.strip()[:90])
    a = stats.setdefault(key, [0.0, 0.0])
    a[0] += inst
    a[1] += samp
tot_i = sum(v[0] for v in stats.values()) or 1
tot_s = sum(v[1] for v in stats.values()) or 1
print(f"total warp inst {tot_i:.3e}, stall samples {tot_s:.0f}")
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{100 * v[1] / tot_s:5.1f}% samp {100 * v[0] / tot_i:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
