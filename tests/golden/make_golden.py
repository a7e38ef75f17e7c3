"""Generate the golden fixtures by running the REAL reference package.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--config-check]

Imports ``linopkit`` from /root/reference/pkg/src (read-only; present only in
the build container, never on the GPU box) and records its outputs on seeded
inputs into ``tests/golden/*.npz``.  The CPU test-suite pins the oracle
(oracle/linop_oracle.py) against these fixtures; the GPU suite checks the
device path against the oracle and against the fixtures.

``--config-check`` additionally runs the reference and the oracle on column
samples of the five BASELINE configs at full transform length and writes the
relative errors to tests/golden/config_check.txt.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(HERE))

import linopkit as lk  # noqa: E402  (the reference)
from make_problems import solver_problems  # noqa: E402


def cn(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)


def gen_kernels():
    out = {}
    for n in list(range(1, 18)) + [32, 100, 128, 1009]:
        rng = np.random.default_rng(n)
        x = cn(rng, (n, 2))
        out[f"dft/n={n}/x"] = x
        out[f"dft/n={n}/fwd"] = lk.dft(x)
        out[f"dft/n={n}/inv"] = lk.dft(x, inverse=True)
    for order in range(0, 11):
        rng = np.random.default_rng(100 + order)
        x = rng.standard_normal((1 << order, 3))
        out[f"fwht/order={order}/x"] = x
        out[f"fwht/order={order}/y"] = lk.fwht(x)
    for n in [1, 2, 3, 5, 8, 17, 64]:
        rng = np.random.default_rng(200 + n)
        c = rng.standard_normal(n)
        x = rng.standard_normal((n, 2))
        out[f"cconv/n={n}/c"] = c
        out[f"cconv/n={n}/x"] = x
        out[f"cconv/n={n}/y"] = lk.circular_convolve(c, x)
    return out


def _fb(out, key, op, x, y):
    out[f"{key}/x"] = x
    out[f"{key}/y"] = y
    out[f"{key}/fwd"] = op.forward(x)
    out[f"{key}/bwd"] = op.backward(y)


def gen_ops():
    out = {}
    # Hadamard: orders 0..12, real and int32 inputs (reference returns float64)
    for order in range(0, 13):
        rng = np.random.default_rng(300 + order)
        n = 1 << order
        op = lk.Hadamard(order)
        _fb(out, f"hadamard/order={order}", op, rng.standard_normal((n, 3)), rng.standard_normal((n, 3)))
        xi = rng.integers(-100, 101, (n, 3), dtype=np.int32)
        out[f"hadamard_i32/order={order}/x"] = xi
        out[f"hadamard_i32/order={order}/y"] = op.forward(xi)
    # C1 exactly (seeded as SURVEY §8d)
    rng = np.random.default_rng([1710, 1])
    X = rng.standard_normal((1024, 16))
    Xi = rng.integers(-100, 101, (1024, 16), dtype=np.int32)
    op = lk.Hadamard(10)
    out["c1/X"] = X
    out["c1/Xi"] = Xi
    out["c1/fwd"] = op.forward(X)
    out["c1/bwd"] = op.backward(X)
    out["c1/fwd_i32"] = op.forward(Xi)
    # Fourier incl. Bluestein lengths
    for n in [1, 2, 5, 8, 12, 17, 61, 64, 256, 1009, 4096, 5000, 8192]:
        rng = np.random.default_rng(400 + n)
        _fb(out, f"fourier/n={n}", lk.Fourier(n), cn(rng, (n, 2)), cn(rng, (n, 2)))
    # Circulant: real / complex kernels, real / complex inputs
    for n in [1, 2, 3, 4, 7, 8, 12, 64, 256, 1000, 4096, 8192]:
        rng = np.random.default_rng(500 + n)
        c = rng.standard_normal(n)
        _fb(out, f"circulant_rr/n={n}", lk.Circulant(c), rng.standard_normal((n, 2)),
            rng.standard_normal((n, 2)))
        out[f"circulant_rr/n={n}/c"] = c
        cc = cn(rng, n)
        _fb(out, f"circulant_cc/n={n}", lk.Circulant(cc), cn(rng, (n, 2)), cn(rng, (n, 2)))
        out[f"circulant_cc/n={n}/c"] = cc
    # Toeplitz: the reference's 20 random shapes <= 32, then larger shapes
    rng = np.random.default_rng(50)
    shapes = [(int(rng.integers(1, 33)), int(rng.integers(1, 33))) for _ in range(20)]
    shapes += [(300, 200), (200, 300), (3000, 3000)]
    for i, (n, m) in enumerate(shapes):
        r2 = np.random.default_rng(600 + i)
        col = r2.standard_normal(n)
        row = r2.standard_normal(m - 1)
        _fb(out, f"toeplitz/{i}", lk.Toeplitz(col, row), r2.standard_normal((m, 2)),
            r2.standard_normal((n, 2)))
        out[f"toeplitz/{i}/col"] = col
        out[f"toeplitz/{i}/row"] = row
    # Kron (np.kron order) small cases, including the C4 factor types
    for i, (o, f, c) in enumerate([(1, 2, 4), (2, 4, 8), (3, 8, 16)]):
        r2 = np.random.default_rng(700 + i)
        cv = cn(r2, c)
        op = lk.Kron(lk.Hadamard(o), lk.Fourier(f), lk.Circulant(cv))
        n = (1 << o) * f * c
        _fb(out, f"kron/{i}", op, cn(r2, (n, 2)), cn(r2, (n, 2)))
        out[f"kron/{i}/c"] = cv
    # C5 chain at small prime sizes, built in the reference algebra
    for N in [61, 1009]:
        r2 = np.random.default_rng(800 + N)
        d1 = np.exp(2j * np.pi * r2.random(N))
        d2 = np.exp(2j * np.pi * r2.random(N))
        U = cn(r2, (N, 4)) / np.sqrt(N)
        V = cn(r2, (N, 4)) / np.sqrt(N)
        order = (N - 1).bit_length()
        idx = np.arange(N)
        hpad = lk.Partial(lk.Hadamard(order), idx, idx)
        lr = lk.Product(lk.Dense(U), lk.Dense(V.conj().T))
        s = lk.Product(lk.Blocks([[hpad, lr]]), lk.Blocks([[lk.Identity(N)], [lk.Identity(N)]]))
        op = lk.Product(lk.Diagonal(d1), lk.Fourier(N), lk.Diagonal(d2), s)
        _fb(out, f"c5/N={N}", op, cn(r2, (N, 3)), cn(r2, (N, 3)))
        for k, v in dict(d1=d1, d2=d2, U=U, V=V).items():
            out[f"c5/N={N}/{k}"] = v
    return out


def gen_extra():
    """Sparse / Polynomial / Power operators and the solvers."""
    P = solver_problems()
    out = {}
    for name in ("sparse_r", "sparse_c"):
        q = P[name]
        op = lk.Sparse(40, 30, list(zip(q["i"].tolist(), q["j"].tolist(), q["v"].tolist())))
        out[f"{name}/fwd"] = op.forward(q["x"])
        out[f"{name}/bwd"] = op.backward(q["y"])
        out[f"{name}/nnz"] = np.asarray(op.nnz)
        out[f"{name}/footprint"] = np.asarray(op.footprint_bytes())
    rng = np.random.default_rng(9)
    x = rng.standard_normal((64, 2))
    xc = cn(rng, (16, 2))
    c = P["poly_c"]
    out["poly_r/x"], out["poly_c/x"] = x, xc
    pr = lk.Polynomial(lk.Circulant(c), [0.5, -1.0, 0.25])
    pc = lk.Polynomial(lk.Fourier(16), np.array([1.0, 0.5j, -0.25]))
    out["poly_r/fwd"], out["poly_r/bwd"] = pr.forward(x), pr.backward(x)
    out["poly_c/fwd"], out["poly_c/bwd"] = pc.forward(xc), pc.backward(xc)
    pw = lk.Power(lk.Circulant(c), 3)
    out["pow3/fwd"], out["pow3/bwd"] = pw.forward(x), pw.backward(x)
    pf = lk.Power(lk.Fourier(16), 2)
    out["powf/fwd"], out["powf/bwd"] = pf.forward(xc), pf.backward(xc)
    out["pow0/fwd"] = lk.Power(lk.Hadamard(6), 0).forward(x)
    # CG: SPD circulant (hermitian mode), complex HPD circulant, Toeplitz normal equations
    r = lk.cg_solve(lk.Circulant(P["spd_c"]), P["cg_rhs"], lk.SolveOptions(assume_hermitian=True))
    out["cg_spd/x"], out["cg_spd/it"], out["cg_spd/res"], out["cg_spd/conv"] = (
        r.solution, r.iterations, r.residual_norm, r.converged)
    r = lk.cg_solve(lk.Circulant(P["hpd_c"]), P["cg_rhs_c"], lk.SolveOptions(assume_hermitian=True))
    out["cg_hpd/x"], out["cg_hpd/it"], out["cg_hpd/res"], out["cg_hpd/conv"] = (
        r.solution, r.iterations, r.residual_norm, r.converged)
    T = lk.Toeplitz(P["toe_col"], P["toe_row"])
    r = lk.cg_solve(T, P["cg_rhs_t"])
    out["cg_ne/x"], out["cg_ne/it"], out["cg_ne/res"], out["cg_ne/conv"] = (
        r.solution, r.iterations, r.residual_norm, r.converged)
    r = lk.cg_solve(T, P["cg_rhs_t"][:, 0], lk.SolveOptions(max_iterations=3))
    out["cg_lim/x"], out["cg_lim/it"], out["cg_lim/res"], out["cg_lim/conv"] = (
        r.solution, r.iterations, r.residual_norm, r.converged)
    # power iteration
    sp = lk.power_iteration(lk.Circulant(P["spd_c"]), seed=3)
    out["pw_eig/value"], out["pw_eig/vec"], out["pw_eig/it"], out["pw_eig/conv"] = (
        sp.value, sp.vector, sp.iterations, sp.converged)
    sp = lk.power_iteration(T, mode="singular", tol=1e-8, seed=1)
    out["pw_sv/value"], out["pw_sv/vec"], out["pw_sv/it"], out["pw_sv/conv"] = (
        sp.value, sp.vector, sp.iterations, sp.converged)
    # ISTA / OMP on compressed-sensing operators
    Mh = lk.Partial(lk.Hadamard(7), row_indices=P["cs_rows_h"])
    bh = Mh.forward(P["cs_x_h"])
    res = lk.ista(Mh, bh, lk.IstaOptions(lam=0.05, steps=60))
    out["ista_h/x"], out["ista_h/trace"], out["ista_h/alpha"] = res.solution, res.objective_trace, res.step_size
    Mf = lk.Partial(lk.Fourier(64), row_indices=P["cs_rows_f"])
    bf = Mf.forward(P["cs_x_f"])
    res = lk.ista(Mf, bf, lk.IstaOptions(lam=0.02, steps=40, step_size=1.0 / 64))
    out["ista_f/x"], out["ista_f/trace"], out["ista_f/alpha"] = res.solution, res.objective_trace, res.step_size
    o = lk.omp(Mh, bh, 4)
    out["omp_h/support"], out["omp_h/coef"], out["omp_h/x"], out["omp_h/res"] = (
        o.support, o.coefficients, o.solution, o.residual_norm)
    o = lk.omp(Mf, bf, 6, residual_tol=1e-9)
    out["omp_f/support"], out["omp_f/coef"], out["omp_f/x"], out["omp_f/res"] = (
        o.support, o.coefficients, o.solution, o.residual_norm)
    out["soft_r"] = lk.soft_threshold(P["soft_r"], 0.5)
    out["soft_c"] = lk.soft_threshold(P["soft_c"], 0.5)
    return out


def config_check(path):
    """Reference vs oracle on column samples of the full-size configs."""
    from oracle import linop_oracle as orc
    from paper_1710_09578_b200 import configs

    lines = []

    def rel(a, b):
        return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

    def both(name, ref_op, orc_op, x, y):
        t0 = time.perf_counter()
        rf, rb = ref_op.forward(x), ref_op.backward(y)
        t1 = time.perf_counter()
        of, ob = orc.apply(orc_op, x, 0), orc.apply(orc_op, y, 1)
        t2 = time.perf_counter()
        exact = bool(np.array_equal(rf, of) and np.array_equal(rb, ob))
        lines.append(f"{name}: relL2 fwd {rel(of, rf):.3e} bwd {rel(ob, rb):.3e} bit-exact {exact} "
                     f"(reference {t1 - t0:.2f}s, oracle {t2 - t1:.2f}s)")
        print(lines[-1], flush=True)

    w = configs.make(1)
    both("C1 f64", lk.Hadamard(10), orc.hadamard(10), w.X, w.X)
    both("C1 int32", lk.Hadamard(10), orc.hadamard(10), w.extra["Xi"], w.extra["Xi"])
    w = configs.make(2, ncols=1)
    both("C2 (1 col)", lk.Circulant(w.params["c"]), orc.circulant(w.params["c"]), w.X, w.X)
    w = configs.make(3, ncols=8)
    p = w.params
    both("C3 (8 cols)", lk.Toeplitz(p["col"], p["row_rest"]), orc.toeplitz(p["col"], p["row_rest"]), w.X, w.X)
    w = configs.make(4, ncols=1)
    p = w.params
    both("C4 (1 col)", lk.Kron(lk.Hadamard(6), lk.Fourier(128), lk.Circulant(p["c"])),
         orc.kron(orc.hadamard(6), orc.fourier(128), orc.circulant(p["c"])), w.X, w.X)
    w = configs.make(5, ncols=1)
    p = w.params
    N = p["N"]
    idx = np.arange(N)
    hpad = lk.Partial(lk.Hadamard(20), idx, idx)
    lr = lk.Product(lk.Dense(p["U"]), lk.Dense(p["V"].conj().T))
    s = lk.Product(lk.Blocks([[hpad, lr]]), lk.Blocks([[lk.Identity(N)], [lk.Identity(N)]]))
    ref = lk.Product(lk.Diagonal(p["d1"]), lk.Fourier(N), lk.Diagonal(p["d2"]), s)
    both("C5 (1 col)", ref, orc.chain_c5(N, p["d1"], p["d2"], p["U"], p["V"]), w.X, w.X)
    Path(path).write_text("\n".join(lines) + "\n")


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    np.savez_compressed(HERE / "kernels.npz", **gen_kernels())
    np.savez_compressed(HERE / "ops.npz", **gen_ops())
    np.savez_compressed(HERE / "extra.npz", **gen_extra())
    for f in ("kernels.npz", "ops.npz", "extra.npz"):
        print(f, (HERE / f).stat().st_size, "bytes")
    if "--config-check" in sys.argv:
        config_check(HERE / "config_check.txt")
