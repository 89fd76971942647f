"""Per-SASS-line instruction counts of one kernel from an ncu report (source page)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = next(r for r in rows if "Instructions Executed" in r)
ie, src = h.index("Instructions Executed"), h.index("Source")
smp = h.index("Warp Stall Sampling (All Samples)")
items = []
for r in rows[rows.index(h) + 1:]:
    try:
        items.append((int(r[ie] or 0), int(r[smp] or 0), r[src].strip()))
    except (ValueError, IndexError):
        continue
tot = sum(n for n, _, _ in items)
print("total warp instructions", tot)
if top:
    for n, s, t in sorted(items, key=lambda x: -x[0])[:top]:
        print(f"{n:>10d} {s:>6d}  {t}")
else:
    for n, s, t in items:
        print(f"{n:>10d} {s:>6d}  {t}")
