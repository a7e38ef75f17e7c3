"""CPU tests for the SURVEY.md §8(f) rows: the oracle restatements of Sparse,
Polynomial, Power and the solvers pinned against fixtures produced by the
REAL reference (tests/golden/extra.npz, tests/golden/make_golden.py), and the
reference's validation behaviour of the new public API (no device needed)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import linop_oracle as orc

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_problems import solver_problems  # noqa: E402

import paper_1710_09578_b200 as sm  # noqa: E402
from conftest import GOLDEN, rel_l2  # noqa: E402


@pytest.fixture(scope="module")
def G():
    return dict(np.load(GOLDEN / "extra.npz"))


@pytest.fixture(scope="module")
def P():
    return solver_problems()


def test_sparse_oracle(G, P):
    for name in ("sparse_r", "sparse_c"):
        q = P[name]
        op = orc.sparse(40, 30, list(zip(q["i"], q["j"], q["v"])))
        assert rel_l2(orc.apply(op, q["x"], 0), G[f"{name}/fwd"]) < 1e-14
        assert rel_l2(orc.apply(op, q["y"], 1), G[f"{name}/bwd"]) < 1e-14


def test_sparse_host_side(G, P):
    """CSR assembly (sort, duplicate summing) and footprint are host logic."""
    for name in ("sparse_r", "sparse_c"):
        q = P[name]
        op = sm.Sparse(40, 30, list(zip(q["i"].tolist(), q["j"].tolist(), q["v"].tolist())))
        assert op.nnz == int(G[f"{name}/nnz"])
        assert op.footprint_bytes() == int(G[f"{name}/footprint"])
        dense = np.zeros((40, 30), dtype=op.values.dtype)
        np.add.at(dense, (q["i"], q["j"]), q["v"])
        rebuilt = np.zeros_like(dense)
        for r in range(40):
            for k in range(op.row_ptr[r], op.row_ptr[r + 1]):
                rebuilt[r, op.col_idx[k]] += op.values[k]
        assert np.allclose(rebuilt, dense, rtol=0, atol=1e-14)
        assert all(np.all(np.diff(op.col_idx[op.row_ptr[r]:op.row_ptr[r + 1]]) > 0) for r in range(40))
    with pytest.raises(sm.IndexOutOfRange):
        sm.Sparse(3, 3, [(0, 3, 1.0)])
    e = sm.Sparse(4, 5, [])
    assert e.nnz == 0 and e.shape == (4, 5)


def test_polynomial_power_oracle(G, P):
    c = P["poly_c"]
    circ = orc.circulant(c)
    x, xc = G["poly_r/x"], G["poly_c/x"]
    pr = orc.polynomial(circ, [0.5, -1.0, 0.25])
    assert rel_l2(orc.apply(pr, x, 0), G["poly_r/fwd"]) < 1e-13
    assert rel_l2(orc.apply(pr, x, 1), G["poly_r/bwd"]) < 1e-13
    pc = orc.polynomial(orc.fourier(16), np.array([1.0, 0.5j, -0.25]))
    assert rel_l2(orc.apply(pc, xc, 0), G["poly_c/fwd"]) < 1e-13
    assert rel_l2(orc.apply(pc, xc, 1), G["poly_c/bwd"]) < 1e-13
    pw = orc.power(circ, 3)
    assert rel_l2(orc.apply(pw, x, 0), G["pow3/fwd"]) < 1e-13
    pf = orc.power(orc.fourier(16), 2)
    assert rel_l2(orc.apply(pf, xc, 1), G["powf/bwd"]) < 1e-13
    assert np.array_equal(orc.apply(orc.power(orc.hadamard(6), 0), x, 0), G["pow0/fwd"])


def test_solver_oracle_cg(G, P):
    X, its, res, conv = orc.cg_solve(orc.circulant(P["spd_c"]), P["cg_rhs"], assume_hermitian=True)
    assert rel_l2(X, G["cg_spd/x"]) < 1e-12 and np.array_equal(its, G["cg_spd/it"]) and conv.all()
    X, its, res, conv = orc.cg_solve(orc.circulant(P["hpd_c"]), P["cg_rhs_c"], assume_hermitian=True)
    assert rel_l2(X, G["cg_hpd/x"]) < 1e-12 and np.array_equal(its, G["cg_hpd/it"])
    T = orc.toeplitz(P["toe_col"], P["toe_row"])
    X, its, res, conv = orc.cg_solve(T, P["cg_rhs_t"])
    # normal equations square the condition number: rounding-order differences
    # move the stopping iteration by one
    assert rel_l2(X, G["cg_ne/x"]) < 1e-9 and np.max(np.abs(its - G["cg_ne/it"])) <= 2
    x, it, r, ok = orc.cg_solve(T, P["cg_rhs_t"][:, 0], max_iterations=3)
    assert rel_l2(x, G["cg_lim/x"]) < 1e-12 and it == 3 and not ok
    assert abs(r - float(G["cg_lim/res"])) <= 1e-12 * float(G["cg_lim/res"])


def test_solver_oracle_power_ista_omp(G, P):
    v, vec, it, ok = orc.power_iteration(orc.circulant(P["spd_c"]), seed=3)
    assert abs(v - float(G["pw_eig/value"])) < 1e-12 * v and it == int(G["pw_eig/it"]) and ok
    T = orc.toeplitz(P["toe_col"], P["toe_row"])
    v, vec, it, ok = orc.power_iteration(T, mode="singular", tol=1e-8, seed=1)
    assert abs(v - float(G["pw_sv/value"])) < 1e-12 * v and it == int(G["pw_sv/it"])
    Mh = orc.partial(orc.hadamard(7), P["cs_rows_h"])
    bh = orc.apply(Mh, P["cs_x_h"], 0)
    x, tr, a = orc.ista(Mh, bh, 0.05, 60)
    assert rel_l2(x, G["ista_h/x"]) < 1e-10 and rel_l2(tr, G["ista_h/trace"]) < 1e-10
    assert abs(a - float(G["ista_h/alpha"])) < 1e-12 * a
    Mf = orc.partial(orc.fourier(64), P["cs_rows_f"])
    bf = orc.apply(Mf, P["cs_x_f"], 0)
    x, tr, a = orc.ista(Mf, bf, 0.02, 40, step_size=1.0 / 64)
    assert rel_l2(x, G["ista_f/x"]) < 1e-10 and rel_l2(tr, G["ista_f/trace"]) < 1e-10
    s, c, x, r = orc.omp(Mh, bh, 4)
    assert np.array_equal(s, G["omp_h/support"]) and rel_l2(x, G["omp_h/x"]) < 1e-10
    s, c, x, r = orc.omp(Mf, bf, 6, residual_tol=1e-9)
    assert np.array_equal(s, G["omp_f/support"]) and rel_l2(c, G["omp_f/coef"]) < 1e-10
    assert np.array_equal(orc.soft_threshold(P["soft_r"], 0.5), G["soft_r"])
    assert rel_l2(orc.soft_threshold(P["soft_c"], 0.5), G["soft_c"]) < 1e-15


def test_solver_validation_cpu():
    """The reference's argument checks fire before any device work
    (solvers.py:22-34, 37-60, 109-130, 163-181, 208-228, 277-310)."""
    H = sm.Hadamard(3)
    with pytest.raises(sm.NegativeThreshold):
        sm.soft_threshold(np.ones(3), -1.0)
    with pytest.raises(ValueError):
        sm.SolveOptions(relative_tolerance=0)
    with pytest.raises(ValueError):
        sm.SolveOptions(max_iterations=0)
    with pytest.raises(sm.NonSquare):
        sm.cg_solve(sm.Dense(np.ones((2, 3))), np.ones(2))
    with pytest.raises(sm.DimensionMismatch):
        sm.cg_solve(H, np.ones(7))
    with pytest.raises(ValueError):
        sm.IstaOptions(lam=0)
    with pytest.raises(ValueError):
        sm.IstaOptions(lam=1, steps=0)
    with pytest.raises(ValueError):
        sm.ista(H, np.ones((8, 2)), sm.IstaOptions(lam=1))
    with pytest.raises(sm.DimensionMismatch):
        sm.ista(H, np.ones(7), sm.IstaOptions(lam=1))
    with pytest.raises(sm.KOutOfRange):
        sm.omp(H, np.ones(8), 9)
    with pytest.raises(sm.KOutOfRange):
        sm.omp(H, np.ones(8), 0)
    with pytest.raises(ValueError):
        sm.power_iteration(H, mode="bogus")
    with pytest.raises(sm.NonSquare):
        sm.power_iteration(sm.Dense(np.ones((2, 3))))
    with pytest.raises(sm.NonSquare):
        sm.Polynomial(sm.Dense(np.ones((2, 3))), [1, 2])
    with pytest.raises(sm.EmptyInput):
        sm.Polynomial(H, [])
    with pytest.raises(ValueError):
        sm.Power(H, -1)
    assert issubclass(sm.BreakdownError, ArithmeticError)
    p = sm.Polynomial(H, [1, 2j])
    assert p.field is sm.ScalarField.COMPLEX128 and p.footprint_bytes() == 8 + 32 + H.footprint_bytes()
    assert sm.Power(H, 4).footprint_bytes() == 16 + H.footprint_bytes()
    par = sm.Parametric(lambda i, j: i + j, 3, 4, sm.ScalarField.REAL64)
    assert par.shape == (3, 4) and par.footprint_bytes() == 24


def test_selfcheck_dense_definitions():
    """The self-verification zoo's dense matrices (selfcheck.py) agree with the
    oracle's dense materialisations of the same operators."""
    from paper_1710_09578_b200 import selfcheck as sc

    rng = np.random.default_rng(3)
    for order in range(0, 6):
        assert np.array_equal(sc.hadamard_matrix(order), orc.to_dense(orc.hadamard(order)))
    for n in (1, 2, 5, 8, 12):
        assert np.allclose(sc.dft_matrix(n), orc.to_dense(orc.fourier(n)), atol=1e-12)
        c = rng.standard_normal(n)
        assert np.allclose(sc.circulant_matrix(c), orc.to_dense(orc.circulant(c)), atol=1e-12)
    for n, m in ((1, 1), (3, 5), (6, 2), (7, 7)):
        col, rest = rng.standard_normal(n), rng.standard_normal(m - 1)
        assert np.allclose(sc.toeplitz_matrix(col, rest), orc.to_dense(orc.toeplitz(col, rest)), atol=1e-12)
    names = {name for name, _, _ in sc.build_zoo(max_size=16)}
    assert names == {"Dense", "Zero", "Identity", "Diagonal", "Sparse", "Fourier", "Circulant", "Toeplitz",
                     "Parametric", "Hadamard", "Product", "Kron", "Blocks", "BlockDiag", "Partial", "Polynomial",
                     "Power", "Adjoint"}
