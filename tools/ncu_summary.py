"""Key metrics per kernel from an ncu --set full report (for profiles/)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_%peak"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    print("==", name[:110])
    for k, label in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"   {label:22s} {r[i]:>18s} {units[i]}")
    st = sorted(((float(r[hdr.index(h)] or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h in stalls),
                reverse=True)[:int(__import__("os").environ.get("NSTALL", "6"))]
    print("   top stalls:", ", ".join(f"{n}={int(v)}" for v, n in st))
