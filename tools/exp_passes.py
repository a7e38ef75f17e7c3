"""Per-pass device times of one BASELINE config with a given libsmat variant.

    python tools/exp_passes.py CFG [LIB ...]   (LIB: path of a libsmat .so; default the in-tree one)
Prints one line per library: {label: avg ms per launch} over 3 fwd+bwd reps.
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

cfg = int(sys.argv[1])
libs = sys.argv[2:] or [None]
lib = libs[0]
from paper_1710_09578_b200 import _native  # noqa: E402

if lib:
    _native.LIB_PATH = Path(lib).resolve()
from paper_1710_09578_b200 import configs  # noqa: E402
import bench  # noqa: E402

w = configs.make(cfg)
op = configs.operator(cfg, w)
X = torch.from_numpy(np.ascontiguousarray(w.X)).cuda()
K = X.shape[1] if X.dim() == 2 else 1
if np.iscomplexobj(w.X) is False and cfg == 3:
    K = X.shape[1] // 2
plan = op.plan_for(bench.w_dtype(cfg), 0)
stream = torch.cuda.current_stream(0)
Y = op.forward(X)
Z = torch.empty_like(X)
by = {}
R = 4
for _ in range(R):
    for d, (src, dst) in enumerate(((X, Y), (Y, Z))):
        seen = {}
        for lab, t in plan.apply_profiled(d, src, plan.dtype_code, dst, X.shape[1], stream.cuda_stream):
            k = f"{'fb'[d]}:{lab}"
            seen[k] = seen.get(k, 0) + 1
            if seen[k] > 1:
                k += f"#{seen[k]}"
            by.setdefault(k, []).append(t)
res = {k: round(float(np.mean(v[1:])), 4) for k, v in by.items()}
res["_total_ms_per_step"] = round(sum(float(np.mean(v[1:])) for v in by.values()), 4)
Y1 = op.forward(X)
Z1 = op.backward(Y1)
chk = [float(torch.linalg.vector_norm(Y1.to(torch.complex128) if Y1.is_complex() else Y1.double())),
       float(torch.linalg.vector_norm(Z1.to(torch.complex128) if Z1.is_complex() else Z1.double())),
       float((Y1[:, :3].abs().double() * torch.arange(1, Y1.shape[0] + 1, device=Y1.device).double()[:, None]).sum())]
print(json.dumps({"lib": Path(lib).name if lib else "libsmat.so", "cfg": cfg, "passes": res, "chk": chk}))
