"""Small invocations of every device path in one process (smoke(), the C5
blocked chain at a four-step size, fused Partial selections, Sparse wide and
narrow, Polynomial, the solvers) — a quick whole-engine check.  (Meant for
compute-sanitizer, which this GPU pool does not allow.)"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import __graft_entry__ as g  # noqa: E402
import paper_1710_09578_b200 as sm  # noqa: E402

g.smoke()
rng = np.random.default_rng(0)
N = 5003
d1 = np.exp(2j * np.pi * rng.random(N))
d2 = np.exp(2j * np.pi * rng.random(N))
U = (rng.standard_normal((N, 4)) + 1j * rng.standard_normal((N, 4))) / N
V = (rng.standard_normal((N, 4)) + 1j * rng.standard_normal((N, 4))) / N
idx = np.arange(N)
op = sm.Product(sm.Diag(d1), sm.Fourier(N), sm.Diag(d2), sm.Sum(sm.Partial(sm.Hadamard(13), idx, idx), sm.LowRank(U, V)))
X = rng.standard_normal((N, 3)) + 1j * rng.standard_normal((N, 3))
op.backward(op.forward(X))
for base in (sm.Hadamard(10), sm.Fourier(1024)):
    p = sm.Partial(base, rng.choice(1024, 300, replace=False), rng.choice(1024, 500, replace=False))
    p.backward(p.forward(rng.standard_normal((500, 2))))
tri = list(zip(rng.integers(0, 2000, 9000).tolist(), rng.integers(0, 1500, 9000).tolist(), rng.standard_normal(9000).tolist()))
S = sm.Sparse(2000, 1500, tri)
for K in (1, 3, 40):
    S.backward(S.forward(rng.standard_normal((1500, K))))
sm.Polynomial(sm.Circulant(rng.standard_normal(64)), [1.0, 2.0, 0.5]).forward(rng.standard_normal((64, 2)))
spd = np.real(np.fft.ifft(1.0 + np.abs(np.fft.fft(rng.standard_normal(256)))))
sm.cg_solve(sm.Circulant(spd), rng.standard_normal((256, 2)), sm.SolveOptions(assume_hermitian=True, max_iterations=10))
M = sm.Partial(sm.Hadamard(8), row_indices=rng.choice(256, 128, replace=False))
b = M.forward(rng.standard_normal(256))
sm.ista(M, b, sm.IstaOptions(lam=0.1, steps=5))
sm.omp(M, b, 3)
sm.power_iteration(sm.Circulant(spd), max_iter=20)
torch.cuda.synchronize()
print("all paths: ok")
