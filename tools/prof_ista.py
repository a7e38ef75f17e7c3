"""Minimal driver for ncu captures of the device ISTA loop on the reference
bench's ISTA scenario (bench.py --workload ista), a few iterations."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1710_09578_b200 as sm  # noqa: E402

its = int(sys.argv[1]) if len(sys.argv) > 1 else 2
size = 1 << 20
rows, c, xt = bench._ista_problem(size)
op = sm.Product(sm.Partial(sm.Hadamard(21), row_indices=rows), sm.Circulant(c))
b = torch.from_numpy(op.forward(xt)).cuda()
res = sm.ista(op, b, sm.IstaOptions(lam=1.0, steps=its, step_size=1e-3))
torch.cuda.synchronize()
print("ok", float(res.objective_trace[-1]))
