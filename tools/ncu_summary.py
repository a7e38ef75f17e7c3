"""Summarise an ncu report (--set full): per kernel duration, DRAM bytes,
issue/pipe utilisation, occupancy, shared-memory conflicts and top stalls.
usage: python tools/ncu_summary.py report.ncu-rep [name-filter]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
keys = [("gpu__time_duration.sum", "us", 1.0),
        ("dram__bytes_read.sum", "rd", 1.0), ("dram__bytes_write.sum", "wr", 1.0),
        ("launch__registers_per_thread", "regs", 1.0),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1.0),
        ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue%", 1.0),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%", 1.0),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%", 1.0),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankconf", 1.0),
        ("smsp__inst_executed.sum", "inst", 1.0)]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if flt not in name:
        continue
    units = {h: rows[1][i] for i, h in enumerate(hdr)}
    parts = []
    for k, lab, _ in keys:
        if k in hdr:
            parts.append(f"{lab}={r[hdr.index(k)]}{units[k] if lab in ('us','rd','wr') else ''}")
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v > 0.3 and "selected" not in h:
                stalls.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    stalls.sort(reverse=True)
    print(name[:100])
    print("   " + "  ".join(parts))
    print("   stalls/issue: " + ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))
