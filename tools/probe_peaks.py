"""Measured arithmetic peaks of this GPU (smat_probe_peak): DFMA, DMMA,
DFMA+DMMA side by side, FFMA2 — prints one JSON line."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1710_09578_b200 import _native  # noqa: E402

torch.cuda.init()
names = ["dfma_fp64", "dmma_fp64", "dfma_plus_dmma_fp64", "ffma2_fp32"]
out = {n: _native.probe_peak(k, 0) for k, n in enumerate(names)}
out["gpu"] = torch.cuda.get_device_name(0)
out["unit"] = "TFLOP/s"
print(json.dumps(out))
