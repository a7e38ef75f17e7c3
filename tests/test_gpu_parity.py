"""Device parity: libsmat.so (sm_100a) against the golden fixtures and the CPU oracle.

Tolerances (north star): bit-exact for integer FWHT; relative L2 <= 1e-12
for float64/complex128 and <= 1e-5 for float32/complex64 — over the whole
block and, stricter, per column.  float64 FWHT is additionally bit-exact
(same stride-1-first stage order as the reference, kernels.py:181-189).
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_1710_09578_b200 as sm
from conftest import max_col_rel_l2, ref_close, rel_l2
from oracle import linop_oracle as orc

pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.complex64: 1e-5, np.float64: 1e-12, np.complex128: 1e-12}


def _keys(d, prefix):
    return sorted({k.split("/")[1] for k in d if k.startswith(prefix + "/")})


def _close(got, ref, tol, what=""):
    """North-star metrics (relative L2 over the block and per column) and the
    reference's own max|err| / (1 + max|ref|) (tests/oracles.py:82-88), all
    within the precision's tolerance."""
    e1, e2 = rel_l2(got, ref), max_col_rel_l2(got, ref)
    ok3, e3 = ref_close(got, ref, tol)
    assert e1 <= tol and e2 <= tol and ok3, \
        f"{what}: relL2 {e1:.3e} maxcol {e2:.3e} refmetric {e3:.3e} > {tol:.0e}"


def _fb(g, key, op, tol=1e-12, single=False):
    x, y = g[f"{key}/x"], g[f"{key}/y"]
    if single:
        x = x.astype(np.complex64 if np.iscomplexobj(x) else np.float32)
        y = y.astype(np.complex64 if np.iscomplexobj(y) else np.float32)
        tol = 1e-5
    _close(op.forward(x), g[f"{key}/fwd"], tol, key + " fwd")
    _close(op.backward(y), g[f"{key}/bwd"], tol, key + " bwd")


# ------------------------------------------------------------- Hadamard -----
def test_hadamard_golden_bit_exact(golden_ops):
    g = golden_ops
    for o in _keys(g, "hadamard"):
        order = int(o.split("=")[1])
        op = sm.Hadamard(order)
        key = f"hadamard/{o}"
        assert np.array_equal(op.forward(g[f"{key}/x"]), g[f"{key}/fwd"]), key
        assert np.array_equal(op.backward(g[f"{key}/y"]), g[f"{key}/bwd"]), key
        xi = g[f"hadamard_i32/{o}/x"]
        yi = op.forward(xi)
        assert yi.dtype == np.int32
        assert np.array_equal(yi.astype(np.int64), g[f"hadamard_i32/{o}/y"].astype(np.int64)), key


def test_c1_config_exact(golden_ops):
    g = golden_ops
    op = sm.Hadamard(10)
    assert np.array_equal(op.forward(g["c1/X"]), g["c1/fwd"])
    assert np.array_equal(op.backward(g["c1/X"]), g["c1/bwd"])
    yi = op.forward(g["c1/Xi"])
    assert yi.dtype == np.int32
    assert np.array_equal(yi.astype(np.int64), g["c1/fwd_i32"].astype(np.int64))
    # float32 inside tolerance
    _close(op.forward(g["c1/X"].astype(np.float32)), g["c1/fwd"], 1e-5, "c1 f32")


@pytest.mark.parametrize("order", [13, 16, 20])
def test_hadamard_multipass_bit_exact(order):
    rng = np.random.default_rng(order)
    x = rng.standard_normal((1 << order, 3))
    assert np.array_equal(sm.Hadamard(order).forward(x), orc.fwht(x))
    xi = rng.integers(-50, 51, (1 << order, 2)).astype(np.int32)
    assert np.array_equal(sm.Hadamard(order).forward(xi).astype(np.int64),
                          orc.fwht(xi).astype(np.int64))


def test_hadamard_complex_and_involution():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((256, 4)) + 1j * rng.standard_normal((256, 4))
    h = sm.Hadamard(8)
    assert np.array_equal(h.forward(x), orc.fwht(x))
    _close(h.forward(h.forward(x)), 256 * x, 1e-13, "involution")


# -------------------------------------------------- Fourier / Circulant -----
def test_fourier_golden(golden_ops):
    g = golden_ops
    for n in _keys(g, "fourier"):
        op = sm.Fourier(int(n.split("=")[1]))
        _fb(g, f"fourier/{n}", op)
        _fb(g, f"fourier/{n}", op, single=True)


def test_dft_kernel_api(golden_kernels):
    g = golden_kernels
    for n in _keys(g, "dft"):
        x = g[f"dft/{n}/x"]
        _close(sm.dft(x), g[f"dft/{n}/fwd"], 1e-12, n)
        _close(sm.dft(x, inverse=True), g[f"dft/{n}/inv"], 1e-12, n)
    for o in _keys(g, "fwht"):
        assert np.array_equal(sm.fwht(g[f"fwht/{o}/x"]), g[f"fwht/{o}/y"])
    for n in _keys(g, "cconv"):
        got = sm.circular_convolve(g[f"cconv/{n}/c"], g[f"cconv/{n}/x"])
        assert got.dtype == np.float64
        _close(got, g[f"cconv/{n}/y"], 1e-12, n)


def test_circulant_golden(golden_ops):
    g = golden_ops
    for kind in ("circulant_rr", "circulant_cc"):
        for n in _keys(g, kind):
            key = f"{kind}/{n}"
            op = sm.Circulant(g[f"{key}/c"])
            _fb(g, key, op)
            _fb(g, key, op, single=True)
            if kind == "circulant_rr":
                assert op.forward(g[f"{key}/x"]).dtype == np.float64


def test_toeplitz_golden(golden_ops):
    g = golden_ops
    for i in _keys(g, "toeplitz"):
        key = f"toeplitz/{i}"
        op = sm.Toeplitz(g[f"{key}/col"], g[f"{key}/row"])
        _fb(g, key, op)
        _fb(g, key, op, single=True)


def test_kron_golden(golden_ops):
    g = golden_ops
    for i, (o, f, _) in enumerate([(1, 2, 4), (2, 4, 8), (3, 8, 16)]):
        key = f"kron/{i}"
        op = sm.Kron(sm.Hadamard(o), sm.Fourier(f), sm.Circulant(g[f"{key}/c"]))
        _fb(g, key, op)
        _fb(g, key, op, single=True)


def test_c5_chain_golden(golden_ops):
    g = golden_ops
    for n in _keys(g, "c5"):
        key = f"c5/{n}"
        N = int(n.split("=")[1])
        order = (N - 1).bit_length()
        idx = np.arange(N)
        op = sm.Product(sm.Diag(g[f"{key}/d1"]), sm.Fourier(N), sm.Diag(g[f"{key}/d2"]),
                        sm.Sum(sm.Partial(sm.Hadamard(order), idx, idx),
                               sm.LowRank(g[f"{key}/U"], g[f"{key}/V"])))
        _fb(g, key, op)


# ----------------------------------------------------- device tensors -------
def test_torch_cuda_tensors_match_host_path():
    import torch

    rng = np.random.default_rng(7)
    c = rng.standard_normal(4096) + 1j * rng.standard_normal(4096)
    x = (rng.standard_normal((4096, 8)) + 1j * rng.standard_normal((4096, 8))).astype(np.complex64)
    op = sm.Circulant(c)
    host = op.forward(x)
    dev = op.forward(torch.from_numpy(x).cuda())
    assert dev.is_cuda and dev.dtype == torch.complex64
    assert np.array_equal(dev.cpu().numpy(), host)
    back = op.backward(dev)
    _close(back.cpu().numpy(), orc.apply(orc.circulant(c), orc.apply(orc.circulant(c), x), 1), 1e-5, "bwd")
    pinned = torch.from_numpy(x).pin_memory()
    cpu_out = op.forward(pinned)
    assert not cpu_out.is_cuda
    assert np.array_equal(cpu_out.numpy(), host)


def test_vector_input_and_empty_columns():
    op = sm.Fourier(12)
    x = np.arange(12.0)
    y = op.forward(x)
    assert y.shape == (12,) and y.dtype == np.complex128
    _close(y, orc.dft(x), 1e-12, "vec")
    e = op.forward(np.zeros((12, 0)))
    assert e.shape == (12, 0)


def test_large_four_step_fft_and_bluestein():
    rng = np.random.default_rng(11)
    for n in (1 << 14, 1 << 20, 100_003):
        x = rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2))
        op = sm.Fourier(n)
        _close(op.forward(x), orc.dft(x), 1e-12, f"F{n} fwd")
        _close(op.backward(x), orc.dft(x, inverse=True) * n, 1e-12, f"F{n} bwd")
        _close(op.forward(x.astype(np.complex64)), orc.dft(x), 1e-5, f"F{n} c64")


def test_convolution_plan_shapes():
    """The structurally different convolution plans against the oracle:
    single precision Toeplitz with L = 8192 runs one four-step convolution of
    64-point TMA passes (masked pad / truncate), double precision runs the two
    pruned 4096-point halves; a 4096-point complex64 Circulant runs four-step;
    rectangular Toeplitz (rows != cols) exercises the asymmetric masks."""
    rng = np.random.default_rng(21)
    for n, m, dt in ((3000, 3000, np.float32), (3000, 3000, np.float64), (2500, 3100, np.float32),
                     (3100, 2100, np.float64), (1500, 4000, np.float32)):
        col = rng.standard_normal(n)
        row = rng.standard_normal(m - 1)
        op = sm.Toeplitz(col.astype(dt), row.astype(dt))
        ref = orc.toeplitz(col, row)
        x = rng.standard_normal((m, 6))
        y = rng.standard_normal((n, 6))
        tol = TOL[dt]
        _close(op.forward(x.astype(dt)), orc.apply(ref, x), tol, f"T{n}x{m} {dt.__name__} fwd")
        _close(op.backward(y.astype(dt)), orc.apply(ref, y, 1), tol, f"T{n}x{m} {dt.__name__} bwd")
    for n in (4096, 2048, 64, 128):
        c = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        x = rng.standard_normal((n, 8)) + 1j * rng.standard_normal((n, 8))
        op = sm.Circulant(c.astype(np.complex64))
        ref = orc.circulant(c)
        _close(op.forward(x.astype(np.complex64)), orc.apply(ref, x), 1e-5, f"C{n} c64 fwd")
        _close(op.backward(x.astype(np.complex64)), orc.apply(ref, x, 1), 1e-5, f"C{n} c64 bwd")


@pytest.mark.parametrize("K", [1, 3, 8, 64])
def test_four_step_paths_sweep(K):
    """Four-step transforms through every pass variant: blocked intermediate
    (single batch) on the TMA pass (K a multiple of the tile width) and on the
    per-tile pass (K = 1, 3), unblocked intermediates under a Kronecker batch,
    Bluestein with Diag·Fourier·Diag folded into the chirps, both precisions."""
    rng = np.random.default_rng(100 + K)

    def cn(*shape):
        return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)

    cases = []
    for n in (1 << 13, 1 << 15, 1 << 17):
        c = cn(n)
        cases.append((sm.Circulant(c), orc.circulant(c), n))
    for n in (5003, 40_009):
        d1, d2 = np.exp(2j * np.pi * rng.random(n)), np.exp(2j * np.pi * rng.random(n))
        cases.append((sm.Product(sm.Diag(d1), sm.Fourier(n), sm.Diag(d2)),
                      orc.product(orc.diagonal(d1), orc.fourier(n), orc.diagonal(d2)), n))
    c = cn(1 << 13)
    cases.append((sm.Kron(sm.Hadamard(1), sm.Circulant(c)),
                  orc.kron(orc.hadamard(1), orc.circulant(c)), 1 << 14))
    for op, ref, n in cases:
        x = cn(n, K)
        for dt, tol in ((np.complex128, 1e-12), (np.complex64, 1e-5)):
            _close(op.forward(x.astype(dt)), orc.apply(ref, x), tol, f"{op!r} K{K} {dt.__name__} fwd")
            _close(op.backward(x.astype(dt)), orc.apply(ref, x, 1), tol, f"{op!r} K{K} {dt.__name__} bwd")


def test_lowrank_shapes():
    """Rank-r factors U diag(s) V^H against Product(Dense(U), Dense(diag(s) V^H))
    (the reference vehicle, leaves.py:40-46): ranks below / at the 32 limit,
    column counts that are not multiples of the 128-column tiles, row counts
    that are not multiples of the row chunks, with and without s, both
    precisions, forward and adjoint, accumulate (inside a Sum)."""
    rng = np.random.default_rng(33)
    for n, m, r, K in ((1000, 777, 5, 3), (4099, 130, 17, 130), (65, 2000, 32, 200), (3000, 3000, 32, 128)):
        U = (rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))) / np.sqrt(n)
        V = (rng.standard_normal((m, r)) + 1j * rng.standard_normal((m, r))) / np.sqrt(m)
        s = rng.standard_normal(r) + 1j * rng.standard_normal(r)
        for with_s in (False, True):
            op = sm.LowRank(U, V, s) if with_s else sm.LowRank(U, V)
            Vs = V * np.conj(s)[None, :] if with_s else V
            ref = orc.product(orc.dense(U), orc.dense(Vs.conj().T))
            x = rng.standard_normal((m, K)) + 1j * rng.standard_normal((m, K))
            y = rng.standard_normal((n, K)) + 1j * rng.standard_normal((n, K))
            _close(op.forward(x), orc.apply(ref, x), 1e-12, f"LR {n}x{m} r{r} K{K} s{with_s} fwd")
            _close(op.backward(y), orc.apply(ref, y, 1), 1e-12, f"LR {n}x{m} r{r} K{K} s{with_s} bwd")
            _close(op.forward(x.astype(np.complex64)), orc.apply(ref, x), 1e-5, f"LR c64 {n}x{m} r{r}")
        if n == m:
            tot = sm.Sum(sm.Diag(np.ones(n)), sm.LowRank(U, V))
            x = rng.standard_normal((n, K)) + 1j * rng.standard_normal((n, K))
            _close(tot.forward(x), x + orc.apply(orc.product(orc.dense(U), orc.dense(V.conj().T)), x), 1e-12,
                   f"Sum+LR {n} acc")


def test_adjoint_identity_random_ops():
    rng = np.random.default_rng(5)
    ops = [sm.Fourier(1000), sm.Circulant(rng.standard_normal(5000)),
           sm.Toeplitz(rng.standard_normal(300), rng.standard_normal(500)),
           sm.Kron(sm.Hadamard(3), sm.Fourier(5), sm.Diag(rng.standard_normal(7) + 1j))]
    for op in ops:
        x = rng.standard_normal((op.cols, 3)) + 1j * rng.standard_normal((op.cols, 3))
        y = rng.standard_normal((op.rows, 3)) + 1j * rng.standard_normal((op.rows, 3))
        lhs = np.sum(np.conj(y) * op.forward(x))
        rhs = np.sum(np.conj(op.backward(y)) * x)
        assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(op.forward(x)) * np.linalg.norm(y), op


def _random_tree(rng, depth):
    """Random composition tree with its oracle twin (reference tests/test_composites.py:313-398)."""
    if depth == 0:
        kind = rng.choice(["dense", "diagonal", "fourier", "hadamard", "circulant", "toeplitz"])
        n = int(rng.integers(2, 9))
        if kind == "dense":
            m = int(rng.integers(2, 9))
            a = rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))
            return sm.Dense(a), orc.dense(a)
        if kind == "diagonal":
            d = rng.standard_normal(n) + 1j * rng.standard_normal(n)
            return sm.Diagonal(d), orc.diagonal(d)
        if kind == "fourier":
            return sm.Fourier(n), orc.fourier(n)
        if kind == "hadamard":
            o = int(rng.integers(1, 4))
            return sm.Hadamard(o), orc.hadamard(o)
        if kind == "circulant":
            c = rng.standard_normal(n)
            return sm.Circulant(c), orc.circulant(c)
        m = int(rng.integers(2, 9))
        col, row = rng.standard_normal(n), rng.standard_normal(m - 1)
        return sm.Toeplitz(col, row), orc.toeplitz(col, row)
    kind = rng.choice(["product", "kron", "sum", "partial", "adjoint", "blockdiag"])
    child, oc = _random_tree(rng, depth - 1)
    if kind == "product":
        d = rng.standard_normal(child.rows)
        return sm.Product(sm.Diagonal(d), child), orc.product(orc.diagonal(d), oc)
    if kind == "kron":
        d = rng.standard_normal(2)
        return sm.Kron(sm.Diagonal(d), child), orc.kron(orc.diagonal(d), oc)
    if kind == "sum":
        d = rng.standard_normal(child.cols)
        if child.rows == child.cols:
            return sm.Sum(child, sm.Diagonal(d)), orc.sum_(oc, orc.diagonal(d))
        return sm.Sum(child, child), orc.sum_(oc, oc)
    if kind == "partial":
        rows = rng.integers(0, child.rows, size=max(1, child.rows // 2))
        return sm.Partial(child, row_indices=rows), orc.partial(oc, rows=rows)
    if kind == "blockdiag":
        other, oo = _random_tree(rng, 0)
        return sm.BlockDiag(child, other), _orc_blockdiag(oc, oo)
    return sm.Adjoint(child), (oc[1], oc[0], oc[3], oc[2], oc[4])


def _orc_blockdiag(a, b):
    def fwd(x):
        return np.concatenate([a[0](x[: a[3]]), b[0](x[a[3]:])])

    def bwd(y):
        return np.concatenate([a[1](y[: a[2]]), b[1](y[a[2]:])])

    return (fwd, bwd, a[2] + b[2], a[3] + b[3], a[4] and b[4])


def test_fifty_random_trees():
    rng = np.random.default_rng(2024)
    for trial in range(50):
        op, oc = _random_tree(rng, int(rng.integers(1, 4)))
        x = rng.standard_normal((op.cols, 2)) + 1j * rng.standard_normal((op.cols, 2))
        y = rng.standard_normal((op.rows, 2)) + 1j * rng.standard_normal((op.rows, 2))
        _close(op.forward(x), orc.apply(oc, x, 0), 1e-12, f"tree {trial} fwd {op!r}")
        _close(op.backward(y), orc.apply(oc, y, 1), 1e-12, f"tree {trial} bwd {op!r}")


def test_to_dense_and_blocks():
    rng = np.random.default_rng(9)
    a = rng.standard_normal((3, 4))
    b = rng.standard_normal((3, 2))
    op = sm.Blocks([[sm.Dense(a), sm.Dense(b)], [sm.Zero(2, 4), sm.Identity(2)]])
    ref = np.block([[a, b], [np.zeros((2, 4)), np.eye(2)]])
    _close(op.to_dense(), ref, 1e-13, "blocks dense")
    _close(sm.Hadamard(1).to_dense(), [[1, 1], [1, -1]], 0, "H1")
    _close(sm.Fourier(2).to_dense(), [[1, 1], [1, -1]], 1e-15, "F2")


@pytest.mark.parametrize("N,K", [(5003, 4), (5003, 3), (70001, 8), (70001, 64)])
def test_c5_blocked_chain(N, K):
    """The C5 chain at four-step sizes compiles into the blocked chain
    (DFSumNode: blocked Sum intermediate, split Hadamard, row-mapped LowRank)
    and matches the oracle forward and backward to 1e-12."""
    rng = np.random.default_rng(N + K)
    d1 = np.exp(2j * np.pi * rng.random(N))
    d2 = np.exp(2j * np.pi * rng.random(N))
    U = (rng.standard_normal((N, 32)) + 1j * rng.standard_normal((N, 32))) / np.sqrt(2 * N)
    V = (rng.standard_normal((N, 32)) + 1j * rng.standard_normal((N, 32))) / np.sqrt(2 * N)
    idx = np.arange(N)
    order = (N - 1).bit_length()
    op = sm.Product(sm.Diag(d1), sm.Fourier(N), sm.Diag(d2),
                    sm.Sum(sm.Partial(sm.Hadamard(order), idx, idx), sm.LowRank(U, V)))
    assert "BlockedChain" in op.plan_for(np.complex128).describe()
    oo = orc.chain_c5(N, d1, d2, U, V)
    X = (rng.standard_normal((N, K)) + 1j * rng.standard_normal((N, K))) / np.sqrt(2)
    _close(op.forward(X), orc.apply(oo, X, 0), 1e-12, f"C5 blocked fwd N={N} K={K}")
    _close(op.backward(X), orc.apply(oo, X, 1), 1e-12, f"C5 blocked bwd N={N} K={K}")


@pytest.mark.parametrize("K", [8, 12])
def test_1024_point_outer_passes(K):
    """Bluestein length 2^20 = 1024 x 1024: the complex128 1024-point masked
    twiddle passes (per-thread stores, landing buffer refilled from inside the
    transform, epilogue slice on its own barrier) at a second geometry than
    C5's — plain Diag·Fourier·Diag (no fused Walsh-Hadamard, patch rows) and
    the blocked chain (fused input / output Walsh-Hadamard, N1 = 16 x 64) —
    plus the spectrum pass's deferred refill at 1024 points."""
    N = 300_007
    rng = np.random.default_rng(N + K)
    d1 = np.exp(2j * np.pi * rng.random(N))
    d2 = np.exp(2j * np.pi * rng.random(N))
    X = (rng.standard_normal((N, K)) + 1j * rng.standard_normal((N, K))) / np.sqrt(2)
    op = sm.Product(sm.Diag(d1), sm.Fourier(N), sm.Diag(d2))
    ref = orc.product(orc.diagonal(d1), orc.fourier(N), orc.diagonal(d2))
    _close(op.forward(X), orc.apply(ref, X, 0), 1e-12, f"DFD fwd N={N} K={K}")
    _close(op.backward(X), orc.apply(ref, X, 1), 1e-12, f"DFD bwd N={N} K={K}")
    U = (rng.standard_normal((N, 32)) + 1j * rng.standard_normal((N, 32))) / np.sqrt(2 * N)
    V = (rng.standard_normal((N, 32)) + 1j * rng.standard_normal((N, 32))) / np.sqrt(2 * N)
    idx = np.arange(N)
    order = (N - 1).bit_length()
    chain = sm.Product(sm.Diag(d1), sm.Fourier(N), sm.Diag(d2),
                       sm.Sum(sm.Partial(sm.Hadamard(order), idx, idx), sm.LowRank(U, V)))
    assert "BlockedChain" in chain.plan_for(np.complex128).describe()
    oo = orc.chain_c5(N, d1, d2, U, V)
    Yc, Zc = chain.forward(X), chain.backward(X)
    _close(Yc, orc.apply(oo, X, 0), 1e-12, f"chain fwd N={N} K={K}")
    _close(Zc, orc.apply(oo, X, 1), 1e-12, f"chain bwd N={N} K={K}")
    # (a refill racing with a buffer still in use would show as run-to-run
    # differences: the passes are deterministic, so repeats are bit-identical)
    for _ in range(3):
        assert np.array_equal(chain.forward(X), Yc) and np.array_equal(chain.backward(X), Zc)


@pytest.mark.parametrize("order,K", [(6, 1), (10, 3), (13, 2), (21, 1)])
def test_partial_hadamard_fused_selection(order, K):
    """Partial(Hadamard) with unique arbitrary row / column selections runs as
    FWHT passes with the selection fused (int32 row maps: gather on store,
    scatter on load) and matches the oracle's scatter -> FWHT -> gather."""
    rng = np.random.default_rng(order * 10 + K)
    n = 1 << order
    rows = rng.choice(n, size=n // 2, replace=False)
    cols = rng.choice(n, size=n // 3 + 1, replace=False)
    for r, c in ((rows, None), (None, cols), (rows, cols)):
        op = sm.Partial(sm.Hadamard(order), r, c)
        assert "SelectedHadamard" in op.plan_for(np.float64).describe()
        oo = orc.partial(orc.hadamard(order), r, c)
        x = rng.standard_normal((op.cols, K))
        y = rng.standard_normal((op.rows, K))
        _close(op.forward(x), orc.apply(oo, x, 0), 1e-12, f"partial H fwd order={order}")
        _close(op.backward(y), orc.apply(oo, y, 1), 1e-12, f"partial H bwd order={order}")
        if order <= 10:  # accumulate path (inside a Sum)
            s = sm.Sum(op, sm.Dense(np.ones((op.rows, op.cols)) * 0.5))
            so = orc.sum_(oo, orc.dense(np.ones((op.rows, op.cols)) * 0.5))
            _close(s.forward(x), orc.apply(so, x, 0), 1e-12, "partial H in Sum")


@pytest.mark.parametrize("N,K", [(5003, 4), (70001, 8)])
def test_c5_blocked_chain_with_singular_values(N, K):
    """LowRank(U, V, s) inside the blocked chain: diag(s) folded into the
    cuBLAS expansion factors (plain and blocked-row copies) at plan time."""
    rng = np.random.default_rng(N * 3 + K)
    d1 = np.exp(2j * np.pi * rng.random(N))
    d2 = np.exp(2j * np.pi * rng.random(N))
    U = (rng.standard_normal((N, 8)) + 1j * rng.standard_normal((N, 8))) / np.sqrt(2 * N)
    V = (rng.standard_normal((N, 8)) + 1j * rng.standard_normal((N, 8))) / np.sqrt(2 * N)
    s = rng.standard_normal(8) + 1j * rng.standard_normal(8)
    idx = np.arange(N)
    order = (N - 1).bit_length()
    op = sm.Product(sm.Diag(d1), sm.Fourier(N), sm.Diag(d2),
                    sm.Sum(sm.Partial(sm.Hadamard(order), idx, idx), sm.LowRank(U, V, s)))
    oo = orc.product(orc.diagonal(d1), orc.fourier(N), orc.diagonal(d2),
                     orc.sum_(orc.hadamard_padded(N), orc.lowrank(U, V, s)))
    X = (rng.standard_normal((N, K)) + 1j * rng.standard_normal((N, K))) / np.sqrt(2)
    _close(op.forward(X), orc.apply(oo, X, 0), 1e-12, "C5 chain with s fwd")
    _close(op.backward(X), orc.apply(oo, X, 1), 1e-12, "C5 chain with s bwd")
    lr = sm.LowRank(U, V, s)
    _close(lr.forward(X), orc.apply(orc.lowrank(U, V, s), X, 0), 1e-12, "LowRank with s fwd")
    _close(lr.backward(X), orc.apply(orc.lowrank(U, V, s), X, 1), 1e-12, "LowRank with s bwd")


@pytest.mark.parametrize("n,K,dt", [(64, 1, np.complex128), (1024, 3, np.complex128), (4096, 2, np.complex64),
                                    (8192, 2, np.complex128)])
def test_partial_fourier_fused_selection(n, K, dt):
    """Partial(Fourier(n)) — the partial-Fourier compressed-sensing operator —
    with unique selections: one FFT tile pass with the selection fused into
    its load / store (n <= 4096); longer transforms keep the generic
    scatter / gather path.  Matches the oracle."""
    rng = np.random.default_rng(n + K)
    rows = rng.choice(n, size=n // 3, replace=False)
    cols = rng.choice(n, size=n // 2, replace=False)
    tol = 1e-5 if dt == np.complex64 else 1e-12
    for r, c in ((rows, None), (None, cols), (rows, cols)):
        op = sm.Partial(sm.Fourier(n), r, c)
        if n <= 4096:
            assert "SelectedFourier" in op.plan_for(dt).describe()
        oo = orc.partial(orc.fourier(n), r, c)
        x = (rng.standard_normal((op.cols, K)) + 1j * rng.standard_normal((op.cols, K))).astype(dt)
        y = (rng.standard_normal((op.rows, K)) + 1j * rng.standard_normal((op.rows, K))).astype(dt)
        _close(op.forward(x), orc.apply(oo, x, 0), tol, f"partial F fwd n={n}")
        _close(op.backward(y), orc.apply(oo, y, 1), tol, f"partial F bwd n={n}")
        xr = rng.standard_normal((op.cols, K))  # real input to the complex operator
        _close(op.forward(xr), orc.apply(oo, xr, 0), 1e-12, f"partial F real fwd n={n}")


def test_c5_chain_random_sizes():
    """The C5-type chain over a spread of lengths (Bluestein single-tile and
    four-step, blocked chain taken or not) and column counts: fwd / bwd vs the
    oracle at 1e-12, and the adjoint identity."""
    rng = np.random.default_rng(1710_5)
    for N in (97, 1031, 4099, 12289, 40009, 131101):
        K = int(rng.integers(1, 7))
        d1 = np.exp(2j * np.pi * rng.random(N))
        d2 = np.exp(2j * np.pi * rng.random(N))
        r = int(rng.integers(1, 33))
        U = (rng.standard_normal((N, r)) + 1j * rng.standard_normal((N, r))) / np.sqrt(2 * N)
        V = (rng.standard_normal((N, r)) + 1j * rng.standard_normal((N, r))) / np.sqrt(2 * N)
        idx = np.arange(N)
        order = (N - 1).bit_length()
        op = sm.Product(sm.Diag(d1), sm.Fourier(N), sm.Diag(d2),
                        sm.Sum(sm.Partial(sm.Hadamard(order), idx, idx), sm.LowRank(U, V)))
        oo = orc.chain_c5(N, d1, d2, U, V)
        X = rng.standard_normal((N, K)) + 1j * rng.standard_normal((N, K))
        Y = rng.standard_normal((N, K)) + 1j * rng.standard_normal((N, K))
        fx, by = op.forward(X), op.backward(Y)
        _close(fx, orc.apply(oo, X, 0), 1e-12, f"C5-type fwd N={N} K={K} r={r}")
        _close(by, orc.apply(oo, Y, 1), 1e-12, f"C5-type bwd N={N} K={K} r={r}")
        lhs, rhs = np.vdot(Y, fx), np.vdot(by, X)
        assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(X) * np.linalg.norm(Y) * np.sqrt(N)


# ------------------------------------------------ strided views (ABI v3) ----
def _c5_small(N, seed):
    rng = np.random.default_rng(seed)
    d1 = np.exp(2j * np.pi * rng.random(N))
    d2 = np.exp(2j * np.pi * rng.random(N))
    U = (rng.standard_normal((N, 32)) + 1j * rng.standard_normal((N, 32))) / np.sqrt(2 * N)
    V = (rng.standard_normal((N, 32)) + 1j * rng.standard_normal((N, 32))) / np.sqrt(2 * N)
    idx = np.arange(N)
    order = (N - 1).bit_length()
    op = sm.Product(sm.Diag(d1), sm.Fourier(N), sm.Diag(d2),
                    sm.Sum(sm.Partial(sm.Hadamard(order), idx, idx), sm.LowRank(U, V)))
    return op, orc.chain_c5(N, d1, d2, U, V), rng


def test_strided_column_slices_in_place():
    """A column slice of a wider row-major block (leading dimension > ncols)
    goes through smat_apply with its leading dimension: no staging copy (the
    workspace is the dense one) and the same result as the dense block — for
    the four-step convolution (C2 path) and the blocked C5 chain."""
    import torch

    from paper_1710_09578_b200 import _native

    rng = np.random.default_rng(77)
    n = 1 << 16
    c = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    big = torch.from_numpy(rng.standard_normal((n, 16)) + 1j * rng.standard_normal((n, 16))).cuda()
    view = big[:, 3:9]
    assert not view.is_contiguous()
    op = sm.Circulant(c)
    plan = op.plan_for(np.complex128)
    for d in (0, 1):
        assert plan.workspace_bytes(d, 6, 16, 0, _native.ROW_MAJOR) == plan.workspace_bytes(d, 6)
    oc = orc.circulant(c)
    xs = view.cpu().numpy()
    _close(op.forward(view).cpu().numpy(), orc.apply(oc, xs, 0), 1e-12, "strided circulant fwd")
    _close(op.backward(view).cpu().numpy(), orc.apply(oc, xs, 1), 1e-12, "strided circulant bwd")

    N = 70001
    op5, o5, rng = _c5_small(N, 5)
    big = torch.from_numpy(rng.standard_normal((N, 12)) + 1j * rng.standard_normal((N, 12))).cuda()
    view = big[:, 5:12]
    plan = op5.plan_for(np.complex128)
    for d in (0, 1):
        assert plan.workspace_bytes(d, 7, 12, 0, _native.ROW_MAJOR) == plan.workspace_bytes(d, 7)
    xs = view.cpu().numpy()
    _close(op5.forward(view).cpu().numpy(), orc.apply(o5, xs, 0), 1e-12, "strided C5 fwd")
    _close(op5.backward(view).cpu().numpy(), orc.apply(o5, xs, 1), 1e-12, "strided C5 bwd")


def test_column_major_and_staged_views():
    """Column-major blocks (a transposed tensor) and strided views that a
    plan cannot address in place are staged through the workspace with one
    device copy each way; numpy strided arrays take pitched host copies."""
    import torch

    rng = np.random.default_rng(78)
    n, K = 1 << 14, 5
    xt = torch.from_numpy(rng.standard_normal((K, n)) + 1j * rng.standard_normal((K, n))).cuda()
    x = xt.t()  # (n, K) column-major view
    for op, oo in ((sm.Hadamard(14), orc.hadamard(14)), (sm.Fourier(n), orc.fourier(n)),
                   (sm.Kron(sm.Hadamard(4), sm.Fourier(1 << 10)), orc.kron(orc.hadamard(4), orc.fourier(1 << 10)))):
        xs = x.cpu().numpy()
        _close(op.forward(x).cpu().numpy(), orc.apply(oo, xs, 0), 1e-12, f"col-major {op!r} fwd")
        _close(op.backward(x).cpu().numpy(), orc.apply(oo, xs, 1), 1e-12, f"col-major {op!r} bwd")
        wide = x.contiguous()
        big = torch.zeros((n, 2 * K), dtype=wide.dtype, device="cuda")
        big[:, 1:1 + K] = wide
        sl = big[:, 1:1 + K]
        _close(op.forward(sl).cpu().numpy(), orc.apply(oo, xs, 0), 1e-12, f"slice {op!r} fwd")
    # numpy host arrays: a column slice and a Fortran-order block
    A = rng.standard_normal((n, 9))
    oo = orc.hadamard(14)
    _close(sm.Hadamard(14).forward(A[:, 2:7]), orc.apply(oo, A[:, 2:7], 0), 0, "numpy slice")
    F = np.asfortranarray(A)
    _close(sm.Hadamard(14).forward(F), orc.apply(oo, A, 0), 0, "numpy fortran")


def test_toeplitz_single_precision_shapes():
    """Single precision Toeplitz with L = 8192 (the four-step convolution):
    square and rectangular shapes, the 4096-row edge, complex64 data, an odd
    real column count (no column-pair packing), accumulation inside a Sum, and
    a strided column slice (leading dimension, transformed in place) against
    the oracle."""
    import torch

    rng = np.random.default_rng(31)
    for n, m, K, cplx in ((3000, 3000, 64, False), (4096, 4096, 6, False), (4000, 1500, 10, False),
                          (1500, 4000, 4, False), (4096, 2, 2, False), (3000, 3000, 5, True),
                          (2500, 3100, 3, True), (3000, 3000, 7, False)):
        col = rng.standard_normal(n) + (1j * rng.standard_normal(n) if cplx else 0)
        row = rng.standard_normal(m - 1) + (1j * rng.standard_normal(m - 1) if cplx else 0)
        dt = np.complex64 if cplx else np.float32
        op = sm.Toeplitz(col.astype(dt), row.astype(dt))
        ref = orc.toeplitz(col, row)
        x = rng.standard_normal((m, K)) + (1j * rng.standard_normal((m, K)) if cplx else 0)
        y = rng.standard_normal((n, K)) + (1j * rng.standard_normal((n, K)) if cplx else 0)
        _close(op.forward(x.astype(dt)), orc.apply(ref, x), 1e-5, f"T{n}x{m} K{K} fwd")
        _close(op.backward(y.astype(dt)), orc.apply(ref, y, 1), 1e-5, f"T{n}x{m} K{K} bwd")
    # accumulation: Toeplitz + Diagonal
    n = 3000
    col, row = rng.standard_normal(n), rng.standard_normal(n - 1)
    d = rng.standard_normal(n)
    op = sm.Toeplitz(col.astype(np.float32), row.astype(np.float32)) + sm.Diagonal(d.astype(np.float32))
    x = rng.standard_normal((n, 8))
    want = orc.apply(orc.toeplitz(col, row), x) + d[:, None] * x
    _close(op.forward(x.astype(np.float32)), want, 1e-5, "Toeplitz + Diagonal")
    # strided column slice of a wider device block: transformed in place
    t = sm.Toeplitz(col.astype(np.float32), row.astype(np.float32))
    big = rng.standard_normal((n, 40)).astype(np.float32)
    Xd = torch.from_numpy(big).cuda()[:, 4:36]
    got = t.forward(Xd).cpu().numpy()
    _close(got, orc.apply(orc.toeplitz(col, row), big[:, 4:36].astype(np.float64)), 1e-5, "strided slice")
