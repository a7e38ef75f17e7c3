"""Seeded solver / §8(f) problems shared by make_golden.py and the tests.

numpy only: importable on the GPU box (no reference package needed).
"""

from __future__ import annotations

import numpy as np


def cn(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)


def solver_problems():
    """Seeded problems shared by gen_extra() and the tests (numpy only)."""
    rng = np.random.default_rng(1710_8)
    P = {}
    # sparse triplets with duplicates, real and complex values
    for name, cplx in (("sparse_r", False), ("sparse_c", True)):
        i = rng.integers(0, 40, 120)
        j = rng.integers(0, 30, 120)
        i[:10] = i[10:20]
        j[:10] = j[10:20]
        v = cn(rng, 120) if cplx else rng.standard_normal(120)
        P[name] = dict(i=i, j=j, v=v, x=rng.standard_normal((30, 3)), y=cn(rng, (40, 3)))
    # symmetric positive definite real circulant, Hermitian PD complex circulant
    n = 128
    s = 1.0 + np.abs(rng.standard_normal(n))
    s = 0.5 * (s + np.roll(s[::-1], 1))
    P["spd_c"] = np.real(np.fft.ifft(s))
    P["hpd_c"] = np.fft.ifft(1.0 + np.abs(rng.standard_normal(64)))
    P["cg_rhs"] = rng.standard_normal((n, 4))
    P["cg_rhs_c"] = cn(rng, (64, 2))
    col = rng.standard_normal(60)
    col[0] = 10.0
    P["toe_col"] = col
    P["toe_row"] = rng.standard_normal(59)
    P["cg_rhs_t"] = rng.standard_normal((60, 2))
    # compressed sensing: partial Hadamard / partial Fourier with sparse truth
    P["cs_rows_h"] = np.sort(rng.choice(128, 64, replace=False))
    xt = np.zeros(128)
    xt[rng.choice(128, 4, replace=False)] = rng.standard_normal(4) + np.sign(rng.standard_normal(4))
    P["cs_x_h"] = xt
    P["cs_rows_f"] = np.sort(rng.choice(64, 32, replace=False))
    xf = np.zeros(64, dtype=complex)
    xf[rng.choice(64, 3, replace=False)] = cn(rng, 3) * 2
    P["cs_x_f"] = xf
    P["soft_r"] = rng.standard_normal(50)
    P["soft_c"] = cn(rng, 50)
    P["poly_c"] = rng.standard_normal(64)
    return P
