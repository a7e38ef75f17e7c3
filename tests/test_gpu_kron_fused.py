"""The two-pass Kron(Hadamard(6), A, B) plan (KronNode::run_fused): H_64 split
as H_8 (x) H_8 over the passes of the two FFT factors, each half running
across warp-shuffle lanes of a 4- or 8-column x 8-Hadamard-row tile.

Parity against the CPU oracle (np.kron index order, reference
composites.py:96-107) over every column, forward and backward, for the
factor orders and widths that take the fused path, plus shapes that must
fall back to the mode-wise passes (column counts not a multiple of 8,
complex128, other Hadamard orders) — same results either way.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_1710_09578_b200 as sm
from conftest import max_col_rel_l2
from oracle import linop_oracle as orc

pytestmark = pytest.mark.gpu


def _cplx(rng, shape, dt=np.complex64):
    return ((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)).astype(dt)


def _cuda(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _check(op, oop, X, tol):
    Y = op.forward(_cuda(X)).cpu().numpy()
    Z = op.backward(_cuda(X)).cpu().numpy()
    assert max_col_rel_l2(Y, orc.apply(oop, X, 0)) <= tol
    assert max_col_rel_l2(Z, orc.apply(oop, X, 1)) <= tol


@pytest.mark.parametrize("a_kind,b_kind", [("F128", "C256"), ("F256", "C128"), ("C128", "F128")])
@pytest.mark.parametrize("K", [8, 24])
def test_kron_hadamard_fused_two_passes(a_kind, b_kind, K):
    rng = np.random.default_rng([1710, K, len(a_kind + b_kind)])

    def leaf(kind):
        n = int(kind[1:])
        if kind[0] == "F":
            return sm.Fourier(n), orc.fourier(n)
        c = _cplx(rng, n)
        return sm.Circulant(c), orc.circulant(c)

    (a, oa), (b, ob) = leaf(a_kind), leaf(b_kind)
    op = sm.Kron(sm.Hadamard(6), a, b)
    oop = orc.kron(orc.hadamard(6), oa, ob)
    plan = op.plan_for(np.complex64)
    assert plan.launches(0, K) == 2 and plan.launches(1, K) == 2
    X = _cplx(rng, (op.numM, K))
    _check(op, oop, X, 1e-5)


@pytest.mark.parametrize("case", ["K4", "c128", "H5", "H7"])
def test_kron_hadamard_unfused_shapes(case):
    rng = np.random.default_rng([1710, 7, len(case)])
    order, K, dt = {"K4": (6, 4, np.complex64), "c128": (6, 8, np.complex128), "H5": (5, 8, np.complex64),
                    "H7": (7, 8, np.complex64)}[case]
    c = _cplx(rng, 256, dt)
    op = sm.Kron(sm.Hadamard(order), sm.Fourier(128), sm.Circulant(c))
    oop = orc.kron(orc.hadamard(order), orc.fourier(128), orc.circulant(c))
    assert op.plan_for(dt).launches(0, K) == 3
    X = _cplx(rng, (op.numM, K), dt)
    _check(op, oop, X, 1e-5 if dt == np.complex64 else 1e-12)
