"""Minimal driver for ncu captures: a few applies of one BASELINE workload."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1710_09578_b200 import configs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = configs.make(cfg)
op = configs.operator(cfg, w)
X = torch.from_numpy(np.ascontiguousarray(w.X)).cuda()
for _ in range(reps):
    Y = op.forward(X)
    Z = op.backward(Y)
torch.cuda.synchronize()
print("ok", float(Z.abs().sum()))
