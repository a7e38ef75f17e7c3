"""CPU oracle: a numpy restatement of the reference's transform algorithms.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline / ``--impl reference`` leg use it, and only as the checker (or the
timed CPU baseline), never as the thing measured or shipped.

Every function restates the algorithm of the reference package ``linopkit``
(pkg/src/linopkit/, pure Python + numpy, float64/complex128 arithmetic) —
same operation order where bit-exactness matters (FWHT) and the same
numerical method elsewhere (radix-2 DIT FFT after a bit-reversal gather,
Bluestein chirp-z for other lengths, circulant/Toeplitz via FFT).  It is
pinned against outputs of the reference itself: ``tests/golden/*.npz`` were
produced by importing the reference in the build container
(``tests/golden/make_golden.py``), and ``tests/test_oracle.py`` checks this
module against every fixture and against the reference's own known-answer
tests (tests/test_kernels.py, tests/test_leaves.py of the reference).

Like the reference, all arithmetic is float64/complex128 (core.py:63-73):
int32 Walsh-Hadamard inputs come back as exactly-integral float64.
"""

from __future__ import annotations

import functools

import numpy as np

# ------------------------------------------------------------ helpers ------


def _pow2(n: int) -> bool:
    return n >= 1 and not (n & (n - 1))


def _ceil_pow2(n: int) -> int:
    m = 1
    while m < n:
        m *= 2
    return m


def _as2d(x, dtype):
    a = np.asarray(x, dtype=dtype)
    return (a[:, None], True) if a.ndim == 1 else (a, False)


def bitrev_permutation(n: int) -> np.ndarray:
    """Bit-reversed index order of length n (kernels.py:50-56)."""
    bits = n.bit_length() - 1
    perm = np.zeros(n, dtype=np.intp)
    for b in range(bits):
        lo = 1 << b
        perm[lo:2 * lo] = perm[:lo] + (n >> (b + 1))
    return perm


@functools.lru_cache(maxsize=32)
def _stage_twiddles(n: int):
    """Per-stage twiddles exp(-2 pi i k / size), size = 2, 4, ..., n (kernels.py:73-82)."""
    out = []
    size = 2
    while size <= n:
        out.append(np.exp(-2j * np.pi * np.arange(size // 2) / size))
        size *= 2
    return tuple(out)


def fft_radix2(x: np.ndarray) -> np.ndarray:
    """Radix-2 decimation-in-time FFT along axis 0 of a complex (n, k) batch,
    n a power of two (kernels.py:95-109): bit-reversal gather, then log2(n)
    in-place butterfly stages t = hi*w; hi = lo - t; lo += t."""
    n = x.shape[0]
    a = np.ascontiguousarray(x[bitrev_permutation(n)], dtype=np.complex128)
    k = a.shape[1]
    size = 2
    for w in _stage_twiddles(n):
        h = size // 2
        v = a.reshape(n // size, size, k)
        t = v[:, h:, :] * w[None, :, None]
        v[:, h:, :] = v[:, :h, :] - t
        v[:, :h, :] += t
        size *= 2
    return a


@functools.lru_cache(maxsize=16)
def _bluestein_tables(n: int):
    """Chirp w_j = exp(-i pi (j^2 mod 2n) / n) with exact integer reduction,
    padded length m = next_pow2(2n - 1) and the FFT of the wrapped conjugate
    chirp (kernels.py:83-93)."""
    j = np.arange(n, dtype=np.int64)
    chirp = np.exp(-1j * np.pi * ((j * j) % (2 * n)) / n)
    m = _ceil_pow2(2 * n - 1)
    ker = np.zeros(m, dtype=np.complex128)
    ker[:n] = np.conj(chirp)
    if n > 1:
        ker[m - n + 1:] = np.conj(chirp[1:][::-1])
    spec = fft_radix2(ker[:, None])[:, 0]
    return chirp, m, spec


def fft_bluestein(x: np.ndarray) -> np.ndarray:
    """Chirp-z DFT for any n (kernels.py:111-125)."""
    n, k = x.shape
    chirp, m, spec = _bluestein_tables(n)
    buf = np.zeros((m, k), dtype=np.complex128)
    buf[:n] = x * chirp[:, None]
    conv = fft_radix2(buf)
    conv *= spec[:, None]
    conv = np.conj(fft_radix2(np.conj(conv)))
    conv /= m
    return conv[:n] * chirp[:, None]


def _fft_any(x: np.ndarray) -> np.ndarray:
    return fft_radix2(x) if _pow2(x.shape[0]) else fft_bluestein(x)


def dft(x, inverse: bool = False) -> np.ndarray:
    """Unnormalised DFT along axis 0; the inverse includes 1/n
    (kernels.py:127-161)."""
    a, sq = _as2d(x, np.complex128)
    n = a.shape[0]
    if n == 0:
        raise ValueError("cannot transform an empty vector")
    if inverse:
        out = np.conj(_fft_any(np.conj(a)))
        out /= n
    else:
        out = _fft_any(a)
    return out[:, 0] if sq else out


def fwht(x) -> np.ndarray:
    """Sylvester Walsh-Hadamard transform along axis 0 (kernels.py:164-190):
    stages with half-width 1, 2, 4, ... (stride-1 first), each pairing
    (lower, upper) -> (lower + upper, lower - upper).  float64/complex128 out."""
    arr = np.asarray(x)
    n = arr.shape[0]
    if not _pow2(n):
        raise ValueError(f"length {n} is not a power of two")
    dt = np.complex128 if np.iscomplexobj(arr) else np.float64
    a, sq = _as2d(arr, dt)
    a = a.copy()
    k = a.shape[1]
    h = 1
    while h < n:
        v = a.reshape(n // (2 * h), 2, h, k)
        lo = v[:, 0].copy()
        hi = v[:, 1].copy()
        v[:, 0] = lo + hi
        v[:, 1] = lo - hi
        h *= 2
    return a[:, 0] if sq else a


# ----------------------------------------------------------- operators -----
# Each operator is (forward, backward, rows, cols, is_real_field); forward and
# backward take and return 2-D (rows, k) arrays in float64/complex128.


def _result(out, x_real, op_real):
    return out.real.copy() if (x_real and op_real) else out


def hadamard(order: int):
    n = 1 << order
    f = lambda x: fwht(x)  # noqa: E731  (leaves.py:197-201: fwd == bwd)
    return (f, f, n, n, True)


def fourier(n: int):
    """F (leaves.py:171-172) and F^H = n * IDFT (leaves.py:174-175)."""
    fwd = lambda x: dft(np.asarray(x, np.complex128))  # noqa: E731
    bwd = lambda y: dft(np.asarray(y, np.complex128), inverse=True) * n  # noqa: E731
    return (fwd, bwd, n, n, False)


def circulant(c):
    """Circulant from its first column (leaves.py:207-234)."""
    c = np.asarray(c)
    real = not np.iscomplexobj(c)
    spec = dft(c.astype(np.complex128))
    n = c.shape[0]

    def apply(x, s):
        xr = not np.iscomplexobj(x)
        a = dft(np.asarray(x, np.complex128)) * s[:, None]
        return _result(dft(a, inverse=True), xr, real)

    return (lambda x: apply(x, spec), lambda y: apply(y, np.conj(spec)), n, n, real)


def toeplitz(first_col, first_row_rest=()):
    """Toeplitz via a power-of-two circulant embedding (leaves.py:237-290)."""
    col = np.asarray(first_col)
    row = np.asarray(first_row_rest)
    n = col.shape[0]
    m = row.shape[0] + 1
    real = not (np.iscomplexobj(col) or np.iscomplexobj(row))
    L = _ceil_pow2(n + m - 1)
    emb = np.zeros(L, dtype=np.complex128)
    emb[:n] = col
    if m > 1:
        emb[L - (m - 1):] = row[::-1]
    spec = dft(emb)

    def apply(x, s, nin, nout):
        xr = not np.iscomplexobj(x)
        x = np.asarray(x)
        buf = np.zeros((L, x.shape[1]), dtype=np.complex128)
        buf[:nin] = x
        out = dft(dft(buf) * s[:, None], inverse=True)[:nout]
        return _result(out, xr, real)

    return (lambda x: apply(x, spec, m, n), lambda y: apply(y, np.conj(spec), n, m), n, m, real)


def diagonal(d):
    d = np.asarray(d)
    real = not np.iscomplexobj(d)
    n = d.shape[0]
    return (lambda x: d[:, None] * x, lambda y: np.conj(d)[:, None] * y, n, n, real)


def dense(a):
    a = np.asarray(a)
    real = not np.iscomplexobj(a)
    return (lambda x: a @ x, lambda y: np.conj(a).T @ y, a.shape[0], a.shape[1], real)


def lowrank(U, V, s=None):
    """U diag(s) V^H, restated as Product(Dense(U), [Diagonal(s)], Dense(V^H))."""
    U = np.asarray(U)
    V = np.asarray(V)
    sv = np.ones(U.shape[1]) if s is None else np.asarray(s)
    real = not (np.iscomplexobj(U) or np.iscomplexobj(V) or np.iscomplexobj(sv))
    fwd = lambda x: U @ (sv[:, None] * (np.conj(V).T @ x))  # noqa: E731
    bwd = lambda y: V @ (np.conj(sv)[:, None] * (np.conj(U).T @ y))  # noqa: E731
    return (fwd, bwd, U.shape[0], V.shape[0], real)


def identity(n):
    return (lambda x: np.array(x, copy=True), lambda y: np.array(y, copy=True), n, n, True)


def product(*ops):
    """Right-to-left chain (composites.py:49-61)."""

    def fwd(x):
        for op in reversed(ops):
            x = op[0](x)
        return x

    def bwd(y):
        for op in ops:
            y = op[1](y)
        return y

    return (fwd, bwd, ops[0][2], ops[-1][3], all(o[4] for o in ops))


def sum_(*ops):
    fwd = lambda x: functools.reduce(np.add, [o[0](x) for o in ops])  # noqa: E731
    bwd = lambda y: functools.reduce(np.add, [o[1](y) for o in ops])  # noqa: E731
    return (fwd, bwd, ops[0][2], ops[0][3], all(o[4] for o in ops))


def kron(*ops):
    """np.kron index order, first factor slowest (composites.py:70-121),
    restated as mode-wise application on the (m_0, ..., m_{r-1}, k) view."""

    def apply(x, which):
        x = np.asarray(x)
        k = x.shape[1]
        sizes = [op[3] if which == 0 else op[2] for op in ops]
        t = x.reshape(*sizes, k)
        for a in range(len(ops) - 1, -1, -1):
            op = ops[a]
            t = np.moveaxis(t, a, 0)
            shp = t.shape
            flat = t.reshape(shp[0], -1)
            res = op[which](flat)
            t = np.moveaxis(res.reshape((res.shape[0],) + shp[1:]), 0, a)
        return t.reshape(-1, k)

    rows = int(np.prod([o[2] for o in ops]))
    cols = int(np.prod([o[3] for o in ops]))
    return (lambda x: apply(x, 0), lambda y: apply(y, 1), rows, cols, all(o[4] for o in ops))


def partial(base, rows=None, cols=None):
    """Row/column selection (composites.py:239-320): scatter-add, base, gather."""
    r_idx = None if rows is None else np.asarray(rows, dtype=np.intp)
    c_idx = None if cols is None else np.asarray(cols, dtype=np.intp)

    def scatter(idx, x, length):
        full = np.zeros((length, x.shape[1]), dtype=x.dtype)
        np.add.at(full, idx, x)
        return full

    def fwd(x):
        full = x if c_idx is None else scatter(c_idx, np.asarray(x), base[3])
        out = base[0](full)
        return out if r_idx is None else out[r_idx]

    def bwd(y):
        full = y if r_idx is None else scatter(r_idx, np.asarray(y), base[2])
        out = base[1](full)
        return out if c_idx is None else out[c_idx]

    nr = base[2] if r_idx is None else len(r_idx)
    nc = base[3] if c_idx is None else len(c_idx)
    return (fwd, bwd, nr, nc, base[4])


def hadamard_padded(n: int):
    """Leading n x n block of H_{2^ceil(log2 n)}: Partial(Hadamard, arange(n), arange(n))."""
    order = max(0, (n - 1).bit_length())
    idx = np.arange(n)
    return partial(hadamard(order), idx, idx)


def chain_c5(N, d1, d2, U, V):
    """Diag(d1)·Fourier(N)·Diag(d2)·Sum(Hpad(N), LowRank(U, V)) (BASELINE config 5)."""
    return product(diagonal(d1), fourier(N), diagonal(d2), sum_(hadamard_padded(N), lowrank(U, V)))


def apply(op, x, direction: int = 0):
    """Apply an oracle operator to a 1-D or 2-D array (0 = forward, 1 = backward)."""
    a = np.asarray(x)
    a2 = a[:, None] if a.ndim == 1 else a
    if np.iscomplexobj(a2):
        a2 = a2.astype(np.complex128)
    else:
        a2 = a2.astype(np.float64)
    out = op[direction](a2)
    if op[4] and not np.iscomplexobj(a2):
        out = np.real(out) if np.iscomplexobj(out) else out
    return out[:, 0] if a.ndim == 1 else out


def to_dense(op) -> np.ndarray:
    eye = np.eye(op[3], dtype=np.float64 if op[4] else np.complex128)
    return apply(op, eye, 0)


# ------------------------------------------------- §8(f) operators ---------


def sparse(rows, cols, triplets):
    """CSR from (row, col, value) triplets, duplicates summed (leaves.py:100-159);
    forward CSR @ x, backward conj(CSR)^T @ y, as explicit row loops."""
    tri = list(triplets)
    i = np.asarray([t[0] for t in tri], dtype=np.intp)
    j = np.asarray([t[1] for t in tri], dtype=np.intp)
    v = np.asarray([t[2] for t in tri]) if tri else np.zeros(0)
    real = not np.iscomplexobj(v)
    v = v.astype(np.float64 if real else np.complex128)

    def fwd(x):
        out = np.zeros((rows, x.shape[1]), dtype=np.result_type(v.dtype, x.dtype))
        np.add.at(out, i, v[:, None] * x[j])
        return out

    def bwd(y):
        out = np.zeros((cols, y.shape[1]), dtype=np.result_type(v.dtype, y.dtype))
        np.add.at(out, j, np.conj(v)[:, None] * y[i])
        return out

    return (fwd, bwd, rows, cols, real)


def polynomial(base, coeffs):
    """sum_k coeffs[k] base^k by Horner's rule (composites.py:323-365)."""
    c = np.asarray(coeffs)
    c = c.astype(np.complex128 if np.iscomplexobj(c) else np.float64)

    def run(x, which):
        cc = np.conj(c) if which == 1 else c
        out = cc[-1] * x
        for ck in cc[-2::-1]:
            out = base[which](out)
            out = out + ck * x
        return out

    return (lambda x: run(x, 0), lambda y: run(y, 1), base[2], base[3], base[4] and not np.iscomplexobj(c))


def power(base, k: int):
    """k-fold composition (composites.py:368-398)."""

    def run(x, which):
        out = np.array(x, copy=True)
        for _ in range(k):
            out = base[which](out)
        return out

    return (lambda x: run(x, 0), lambda y: run(y, 1), base[2], base[3], base[4])


# ------------------------------------------------------------ solvers ------
# Restatements of pkg/src/linopkit/solvers.py on oracle operators (tuples).


def soft_threshold(x, c):
    """solvers.py:22-34."""
    arr = np.asarray(x)
    shrunk = np.maximum(np.abs(arr) - c, 0.0)
    if not np.iscomplexobj(arr):
        return np.sign(arr) * shrunk
    scale = np.zeros_like(shrunk)
    np.divide(shrunk, np.abs(arr), out=scale, where=arr != 0)
    return arr * scale


def cg_solve(op, y, max_iterations=None, tol=1e-10, assume_hermitian=False):
    """Column-by-column CG (solvers.py:75-160): returns (X, iterations,
    residual norms, converged); raises ArithmeticError on breakdown."""
    rhs = np.asarray(y)
    squeeze = rhs.ndim == 1
    if squeeze:
        rhs = rhs[:, None]
    real = op[4] and not np.iscomplexobj(rhs)
    dtype = np.float64 if real else np.complex128
    max_iter = max_iterations or op[3]
    if assume_hermitian:
        A = lambda v: apply(op, v, 0)  # noqa: E731
        b = rhs.astype(dtype)
    else:
        A = lambda v: apply(op, apply(op, v, 0), 1)  # noqa: E731
        b = apply(op, rhs, 1).astype(dtype)
    k = rhs.shape[1]
    X = np.zeros((op[3], k), dtype=dtype)
    its = np.zeros(k, dtype=int)
    res = np.zeros(k)
    conv = np.zeros(k, dtype=bool)
    for col in range(k):
        bc = b[:, col].copy()
        x = np.zeros_like(bc)
        r = bc.copy()
        p = r.copy()
        rs_old = np.real(np.vdot(r, r))
        n0 = np.sqrt(rs_old)
        if n0 == 0:
            conv[col] = True
            continue
        thr = tol * n0
        done = False
        for it in range(1, max_iter + 1):
            ap = A(p)
            curv = np.real(np.vdot(p, ap))
            if curv <= 1e-14 * np.linalg.norm(p) * np.linalg.norm(ap):
                raise ArithmeticError(f"breakdown at iteration {it}")
            alpha = rs_old / curv
            x = x + alpha * p
            r = r - alpha * ap
            rs_new = np.real(np.vdot(r, r))
            if np.sqrt(rs_new) <= thr:
                its[col], res[col], conv[col], done = it, np.sqrt(rs_new), True, True
                break
            p = r + (rs_new / rs_old) * p
            rs_old = rs_new
        if not done:
            its[col], res[col] = max_iter, np.sqrt(rs_old)
        X[:, col] = x
    if squeeze:
        return X[:, 0], int(its[0]), float(res[0]), bool(conv[0])
    return X, its, res, conv


def power_iteration(op, mode="eigen", tol=1e-9, max_iter=1000, seed=0):
    """solvers.py:277-333: (value, vector, iterations, converged)."""
    rng = np.random.default_rng(seed)
    n = op[3]
    v = rng.standard_normal(n)
    if not op[4]:
        v = v + 1j * rng.standard_normal(n)
    v = v / np.linalg.norm(v)
    f = (lambda u: apply(op, u, 0)) if mode == "eigen" else (lambda u: apply(op, apply(op, u, 0), 1))
    est = 0.0
    for it in range(1, max_iter + 1):
        w = f(v)
        new = float(np.abs(np.vdot(v, w)))
        nw = np.linalg.norm(w)
        if nw == 0:
            return 0.0, v, it, True
        v = w / nw
        if it > 1 and abs(new - est) <= tol * max(new, 1e-300):
            return float(np.sqrt(new) if mode == "singular" else new), v, it, True
        est = new
    return float(np.sqrt(est) if mode == "singular" else est), v, max_iter, False


def ista(op, b, lam, steps=100, step_size=None, seed=0):
    """solvers.py:163-194: (x, objective trace, step size)."""
    rhs = np.asarray(b)
    alpha = step_size
    if alpha is None:
        alpha = 1.0 / (1.01 * power_iteration(op, "singular", 1e-6, 50, seed)[0] ** 2)
    level = lam * alpha
    x = np.zeros(op[3], dtype=np.result_type(rhs.dtype, np.float64 if op[4] else np.complex128))
    trace = np.empty(steps + 1)
    for k in range(steps):
        r = rhs - apply(op, x, 0)
        trace[k] = lam * np.abs(x).sum() + 0.5 * np.real(np.vdot(r, r))
        x = soft_threshold(x + alpha * apply(op, r, 1), level)
    r = rhs - apply(op, x, 0)
    trace[-1] = lam * np.abs(x).sum() + 0.5 * np.real(np.vdot(r, r))
    return x, trace, float(alpha)


def omp(op, b, sparsity, residual_tol=None):
    """solvers.py:208-261: (support, coefficients, solution, residual norm)."""
    rhs = np.asarray(b)
    dtype = np.result_type(rhs.dtype, np.float64 if op[4] else np.complex128)
    rhs = rhs.astype(dtype)
    stop = residual_tol * np.linalg.norm(rhs) if residual_tol is not None else None
    support = []
    cols = np.zeros((op[2], 0), dtype=dtype)
    coeffs = np.zeros(0, dtype=dtype)
    residual = rhs.copy()
    for _ in range(sparsity):
        corr = np.abs(apply(op, residual, 1))
        corr[support] = -1.0
        atom = int(np.argmax(corr))
        support.append(atom)
        unit = np.zeros(op[3], dtype=dtype)
        unit[atom] = 1
        cols = np.hstack([cols, apply(op, unit, 0)[:, None]])
        coeffs = np.linalg.lstsq(cols, rhs, rcond=None)[0]
        residual = rhs - cols @ coeffs
        if stop is not None and np.linalg.norm(residual) <= stop:
            break
    sol = np.zeros(op[3], dtype=dtype)
    sol[support] = coeffs
    return np.asarray(support, dtype=int), coeffs, sol, float(np.linalg.norm(residual))
