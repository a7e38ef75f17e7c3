"""Top SASS instructions by warp-stall samples from an ncu report's source page.
usage: python tools/ncu_hotspots.py report.ncu-rep [launch_index] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) > 3:
        data.append(r)
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and i != si]
tot = sum(float(r[si] or 0) for r in data if len(r) > si)
print(rows[0][1][:120], "total samples", tot)
print("stall columns:", [hdr[i] for i in stall_cols][:40])
ranked = sorted(data, key=lambda r: -float(r[si] or 0) if len(r) > si else 0)[:top]
for r in ranked:
    extra = []
    for i in stall_cols:
        try:
            v = float(r[i])
        except (ValueError, IndexError):
            continue
        if v > 0.05 * float(r[si] or 1) and v > 0:
            extra.append(f"{hdr[i]}={v:.0f}")
    print(f"{float(r[si]):7.0f} {100*float(r[si])/tot:5.1f}%  {r[0][-5:]} {r[1].strip()[:60]:60s} {' '.join(extra[:4])}")
