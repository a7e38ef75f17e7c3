"""Sparse matrix-vector timing for narrow blocks (K = 1, 4): the solvers'
single-vector case of the CSR kernel."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1710_09578_b200 as sm  # noqa: E402

n, per_row = 1 << 20, 16
rng = np.random.default_rng(3)
rows = np.repeat(np.arange(n), per_row)
cols = rng.integers(0, n, n * per_row)
vals = rng.standard_normal(n * per_row)
S = sm.Sparse.__new__(sm.Sparse)
sm.Sparse._from_arrays(S, n, n, rows, cols, vals)
for K in (1, 4, 64):
    x = torch.from_numpy(rng.standard_normal((n, K))).cuda()
    for _ in range(3):
        S.forward(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        y = S.forward(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    ref = None
    if K == 1:
        import scipy.sparse as ssp
        A = ssp.csr_matrix((vals, (rows, cols)), shape=(n, n))
        ref = A @ x.cpu().numpy()
        err = float(np.linalg.norm(y.cpu().numpy() - ref) / np.linalg.norm(ref))
    print(f"K={K}: {ms:.3f} ms per forward" + (f", rel err vs scipy {err:.2e}" if ref is not None else ""))
