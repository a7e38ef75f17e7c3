"""Executed-instruction mix of a kernel per CUDA source line: joins an ncu
source-page CSV (`ncu -i rep --page source --csv --print-source sass`) with
the line table of the kernel's cubin (`nvdisasm -g -c`).

    python tools/instr_mix.py SRC_CSV CUBIN MANGLED_NAME [top]
"""
import collections
import csv
import re
import subprocess
import sys

src, cubin, name = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
start = next(k for k, l in enumerate(dis) if l.startswith("//---") and (".text." + name) in l)
cur, lmap = None, {}
for l in dis[start + 1:]:
    if l.startswith("//---"):
        break
    mm = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if mm:
        cur = (mm.group(1).split("/")[-1], int(mm.group(2)))
        continue
    mm = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if mm and cur:
        lmap[int(mm.group(1), 16)] = cur
rows = list(csv.reader(open(src)))
hi = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
ix = {n: k for k, n in enumerate(rows[hi])}
data = [r for r in rows[hi + 1:] if r and r[0].startswith("0x")]
base = int(data[0][0], 16)
per = collections.defaultdict(lambda: [0.0, 0.0])
ops = collections.Counter()
tot = 0.0
for r in data:
    v = float(r[ix["Instructions Executed"]] or 0)
    tot += v
    op = r[ix["Source"]].split()
    o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
    ops[o] += v
    key = lmap.get(int(r[0], 16) - base, ("?", 0))
    per[key][0] += v
    if o in ("DADD", "DMUL", "DFMA", "FADD", "FMUL", "FFMA", "FFMA2", "FMUL2", "FADD2", "DMMA"):
        per[key][1] += v
print(f"total warp instructions {tot:.4g}")
print("  " + ", ".join(f"{k}:{v / tot * 100:.1f}%" for k, v in ops.most_common(16)))
for k, (v, f) in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"  {k[0]}:{k[1]:<5} {v / tot * 100:5.1f}%  float {f / max(v, 1) * 100:4.0f}%")
