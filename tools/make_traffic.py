"""profiles/traffic.json: DRAM bytes (read + write) per launch of each bench
kernel label, from the ncu launch lists (dram__bytes_{read,write}.sum).

    python tools/make_traffic.py profiles/r01_launches_c{1..5}.csv
"""

import json
import re
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from summarize_launches import load  # noqa: E402


def label(kernel: str):
    m = re.search(r"fft_(?:tma|tile)_kernel<(float2|double2), (\d+)", kernel)
    if m:
        return ("fft_c64_" if m.group(1) == "float2" else "fft_c128_") + m.group(2)
    m = re.search(r"wht_tile_kernel<[^,]+, (\d+)", kernel)
    if m:
        return "wht_" + m.group(1)
    m = re.search(r"wlr_kernel<(\d+),", kernel)
    if m:  # (the C5 chain: N1 = 2048 = 32 (pass a) x 64 (pass b) unit-row groups)
        return {"32": "wht_lowrank_a", "64": "wht_lowrank_b"}.get(m.group(1), "wlr_" + m.group(1))
    if "lr_contract_kernel" in kernel:
        return "lowrank_contract"
    if "lr_expand_kernel" in kernel:
        return "lowrank_expand"
    for k in ("gemm", "point", "gather", "scatter"):
        if f"{k}_kernel" in kernel:
            return k
    return None


def main(paths):
    out = {}
    for p in paths:
        w = re.search(r"c(\d)\.csv$", p).group(1)
        per = {}
        for d in load(p):
            lab = label(d["kernel"])
            if lab:
                per.setdefault(lab, []).append(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0))
        out["c" + w] = {k: float(statistics.median(v)) for k, v in per.items()}
    dst = Path(__file__).resolve().parent.parent / "profiles" / "traffic.json"
    dst.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(dst.read_text())


if __name__ == "__main__":
    main(sys.argv[1:])
