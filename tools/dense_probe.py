"""Dense (Matrix) leaf timing: library GEMM path vs the SIMT tile kernel
(SMAT_LR_BLAS=0 disables cuBLAS)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1710_09578_b200 as sm  # noqa: E402

rng = np.random.default_rng(0)
for n, K, dt in ((4096, 256, np.float64), (4096, 256, np.complex128), (2048, 64, np.float32)):
    A = rng.standard_normal((n, n)).astype(dt)
    op = sm.Dense(A)
    x = torch.from_numpy(rng.standard_normal((n, K)).astype(dt)).cuda()
    for _ in range(3):
        op.forward(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        y = op.backward(op.forward(x))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    fl = 2 * 2 * n * n * K * (4 if np.iscomplexobj(A) else 1)
    print(f"Dense {n}x{n} K={K} {np.dtype(dt).name}: {ms:.3f} ms fwd+bwd, {fl / ms / 1e9:.1f} TFLOP/s")
