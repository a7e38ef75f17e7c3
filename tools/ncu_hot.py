"""Hot SASS instructions of one kernel from `ncu --page source --csv --print-source sass` output.
usage: python tools/ncu_hot.py source.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows if r and r[0].startswith("0x")]
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[ix[S]] or 0) for r in data)
print("total samples", tot, "instructions", len(data))
kinds = ["stall_wait", "stall_short_sb", "stall_barrier", "stall_long_sb", "stall_mio", "stall_math", "stall_lg"]
best = sorted(range(len(data)), key=lambda i: -float(data[i][ix[S]] or 0))[:top]
for i in sorted(best):
    r = data[i]
    st = " ".join(f"{k[6:]}={r[ix[k]]}" for k in kinds if k in ix and r[ix[k]] not in ("0", ""))
    print(f"{i:5d} {r[ix['Source']].strip()[:48]:48s} {r[ix[S]]:>6s}  {st}")
# samples by opcode
from collections import Counter
c = Counter()
for r in data:
    op = r[ix["Source"]].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    c[o.split(".")[0]] += float(r[ix[S]] or 0)
print(c.most_common(16))
