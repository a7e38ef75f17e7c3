"""Every column of the full-size C2, C4 and C5 blocks against the CPU oracle.

The north-star criterion is "relative L2 over the whole block (and, stricter,
the max over columns)"; the config tests in test_gpu_configs.py sample a few
columns, this module checks all of them.  The device computes the whole block
(forward, then backward of the forward result) once; the oracle columns are
fanned out over the host cores (fork: the workers inherit the inputs and the
device results, compare locally and return only the error norms).
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np
import pytest

from oracle import linop_oracle as orc
from paper_1710_09578_b200 import configs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

_S: dict = {}


def _oracle_op(cfg, w):
    p = w.params
    if cfg == 2:
        return orc.circulant(p["c"])
    if cfg == 4:
        return orc.kron(orc.hadamard(p["h_order"]), orc.fourier(p["f_n"]), orc.circulant(p["c"]))
    return orc.chain_c5(p["N"], p["d1"], p["d2"], p["U"], p["V"])


def _column(j):
    op, X, Y, Z = _S["op"], _S["X"], _S["Y"], _S["Z"]
    ry = orc.apply(op, X[:, j:j + 1], 0)[:, 0]
    rz = orc.apply(op, ry[:, None], 1)[:, 0]
    out = []
    for got, ref in ((Y[:, j], ry), (Z[:, j], rz)):
        out.append((float(np.linalg.norm(got - ref) ** 2), float(np.linalg.norm(ref) ** 2)))
    return j, out


def _all_columns(cfg, tol):
    import torch

    import paper_1710_09578_b200 as sm  # noqa: F401

    w = configs.make(cfg)
    op = configs.operator(cfg, w)
    X = torch.from_numpy(np.ascontiguousarray(w.X)).cuda()
    Y = op.forward(X)
    Z = op.backward(Y)
    _S.update(op=_oracle_op(cfg, w), X=w.X, Y=Y.cpu().numpy(), Z=Z.cpu().numpy())
    del X, Y, Z
    torch.cuda.empty_cache()
    K = w.ncols
    procs = max(1, min(K, len(os.sched_getaffinity(0))))
    with mp.get_context("fork").Pool(procs) as pool:
        res = dict(pool.map(_column, range(K)))
    _S.clear()
    for d, name in ((0, "forward"), (1, "backward")):
        num = np.array([res[j][d][0] for j in range(K)])
        den = np.array([res[j][d][1] for j in range(K)])
        block = float(np.sqrt(num.sum() / den.sum()))
        worst = float(np.max(np.sqrt(num / den)))
        assert block <= tol and worst <= tol, f"C{cfg} {name}: block relL2 {block:.3e}, worst column {worst:.3e}"
    return K


@pytest.mark.timeout(900)
def test_c2_every_column():
    assert _all_columns(2, 1e-5) == 64


@pytest.mark.timeout(900)
def test_c4_every_column():
    assert _all_columns(4, 1e-5) == 32


@pytest.mark.timeout(1800)
def test_c5_every_column():
    assert _all_columns(5, 1e-12) == 128
