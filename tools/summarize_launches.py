"""Summarise an ncu launch list (CSV with gpu__time_duration / dram bytes per
launch) into per-kernel totals: launches, device time, DRAM traffic, share.

    python tools/summarize_launches.py gpurun_out/launches_c2.csv [--skip-build]
"""

import csv
import io
import sys
from collections import OrderedDict


def load(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    ii = h.index("ID")
    launches = OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"kernel": r[ki]})
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        if unit in ("nsecond", "ns"):
            v /= 1e3  # -> us
        elif unit in ("usecond", "us"):
            pass
        elif unit in ("msecond", "ms"):
            v *= 1e3
        elif unit == "Mbyte":
            v *= 1e6
        elif unit == "Gbyte":
            v *= 1e9
        elif unit == "Kbyte":
            v *= 1e3
        d[r[mi]] = v
    return list(launches.values())


def short(name):
    return name.split("(")[0].replace("void ", "")[:70]


def main():
    path = sys.argv[1]
    ls = load(path)
    # drop plan-build kernels (twiddle tables, spectra): everything before the
    # first launch of the applies is setup
    setup = ("tw_init_kernel", "c128_to", "chirp_kernel", "bluestein_kernel_fill", "fourstep_perm",
             "split_even_odd", "point_kernel")
    agg = OrderedDict()
    for d in ls:
        k = short(d["kernel"])
        a = agg.setdefault(k, {"n": 0, "us": 0.0, "bytes": 0.0})
        a["n"] += 1
        a["us"] += d.get("gpu__time_duration.sum", 0.0)
        a["bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    total = sum(a["us"] for a in agg.values())
    print(f"{'kernel':72s} {'launches':>8s} {'time_us':>10s} {'share':>6s} {'dram_GB/launch':>14s} {'GB/s':>8s}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        gbl = a["bytes"] / a["n"] / 1e9 if a["n"] else 0
        gbs = a["bytes"] / (a["us"] * 1e-6) / 1e9 if a["us"] else 0
        print(f"{k:72s} {a['n']:8d} {a['us']:10.1f} {a['us'] / total * 100:5.1f}% {gbl:14.4f} {gbs:8.1f}")
    print(f"{'TOTAL':72s} {sum(a['n'] for a in agg.values()):8d} {total:10.1f}")


if __name__ == "__main__":
    main()
