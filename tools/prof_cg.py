"""Minimal driver for ncu captures of the device-resident CG solver: a few
iterations of cg_solve on the normal equations of C2's operator."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1710_09578_b200 as sm  # noqa: E402
from paper_1710_09578_b200 import configs  # noqa: E402

its = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = configs.make(2)
op = sm.Circulant(w.params["c"])
rhs = torch.from_numpy(np.ascontiguousarray(w.X)).cuda().to(torch.complex128)
rep = sm.cg_solve(op, rhs, sm.SolveOptions(max_iterations=its, relative_tolerance=1e-300))
torch.cuda.synchronize()
print("ok", int(np.max(rep.iterations)))
