"""The five BASELINE.json workloads as seeded synthetic inputs.

No public dataset is involved: every array is drawn with
``numpy.random.default_rng([1710, cfg])`` in the order listed, complex
N(0, s^2) meaning s*(a + ib)/sqrt(2) with a, b iid N(0, 1); blocks are
(rows, K) C-contiguous (the reference's layout).  The same arrays feed the
device path and the CPU oracle.

  C1  Hadamard(10), 1024 x 16 float64 (+ int32 in [-100, 100])
  C2  Circulant(2^20, complex64 column), 2^20 x 64 complex64
  C3  Toeplitz 3000 x 3000 float32, 3000 x 4096 float32
  C4  Kron(Hadamard(6), Fourier(128), Circulant(256, complex64)), 2^21 x 32 complex64
  C5  Diag(d1)·Fourier(1,000,003)·Diag(d2)·Sum(Hpad, LowRank32), 1,000,003 x 128 complex128
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

C5_N = 1_000_003


def _cn(rng, shape, sigma=1.0, dtype=np.complex128):
    a = rng.standard_normal(shape)
    b = rng.standard_normal(shape)
    return (sigma * (a + 1j * b) / np.sqrt(2.0)).astype(dtype)


@dataclass
class Workload:
    name: str
    params: dict
    X: np.ndarray
    extra: dict = field(default_factory=dict)

    @property
    def rows(self):
        return self.X.shape[0]

    @property
    def ncols(self):
        return self.X.shape[1]


def make(cfg: int, ncols: int | None = None, n: int | None = None) -> Workload:
    """Seeded inputs of config `cfg` (1..5).  `ncols` keeps the first columns of
    the full draw (same values as the full block); `n` shrinks the transform
    length for small-size parity cases (same distributions)."""
    rng = np.random.default_rng([1710, cfg])
    if cfg == 1:
        order = 10 if n is None else int(n).bit_length() - 1
        N = 1 << order
        X = rng.standard_normal((N, 16))
        Xi = rng.integers(-100, 101, (N, 16), dtype=np.int32)
        w = Workload("C1 Hadamard(10) 1024x16 f64 + int32", {"order": order}, X, {"Xi": Xi})
        if ncols is not None:
            w.X = w.X[:, :ncols]
            w.extra["Xi"] = w.extra["Xi"][:, :ncols]
        return w
    if cfg == 2:
        N = (1 << 20) if n is None else n
        K = 64
        c = _cn(rng, N, dtype=np.complex64)
        X = _cn(rng, (N, K), dtype=np.complex64)
        w = Workload("C2 Circulant 2^20 x 64 c64", {"c": c}, X)
    elif cfg == 3:
        N = 3000 if n is None else n
        K = 4096
        col = rng.standard_normal(N).astype(np.float32)
        row = rng.standard_normal(N).astype(np.float32)
        row[0] = col[0]
        X = rng.standard_normal((N, K)).astype(np.float32)
        w = Workload("C3 Toeplitz 3000x3000 x 4096 f32", {"col": col, "row_rest": row[1:].copy()}, X)
    elif cfg == 4:
        # modes (64, 128, 256); n scales the circulant mode for small cases
        m3 = 256 if n is None else n
        K = 32
        c = _cn(rng, m3, dtype=np.complex64)
        X = _cn(rng, (64 * 128 * m3, K), dtype=np.complex64)
        w = Workload("C4 Kron(H64, F128, C256) 2^21 x 32 c64", {"c": c, "h_order": 6, "f_n": 128}, X)
    elif cfg == 5:
        N = C5_N if n is None else n
        K = 128
        d1 = np.exp(2j * np.pi * rng.random(N))
        d2 = np.exp(2j * np.pi * rng.random(N))
        U = _cn(rng, (N, 32), sigma=1.0 / np.sqrt(N))
        V = _cn(rng, (N, 32), sigma=1.0 / np.sqrt(N))
        X = _cn(rng, (N, K))
        w = Workload("C5 Diag·F(1000003)·Diag·Sum(Hpad, LowRank32) x 128 c128",
                     {"d1": d1, "d2": d2, "U": U, "V": V, "N": N}, X)
    else:
        raise ValueError(f"unknown config {cfg}")
    if ncols is not None:
        w.X = np.ascontiguousarray(w.X[:, :ncols])
    return w


def operator(cfg: int, w: Workload):
    """The device operator of config `cfg` built from the workload params."""
    from . import (Circulant, Diag, Fourier, Hadamard, Kron, LowRank, Partial, Product, Sum,
                   Toeplitz)

    p = w.params
    if cfg == 1:
        return Hadamard(p["order"])
    if cfg == 2:
        return Circulant(p["c"])
    if cfg == 3:
        return Toeplitz(p["col"], p["row_rest"])
    if cfg == 4:
        return Kron(Hadamard(p["h_order"]), Fourier(p["f_n"]), Circulant(p["c"]))
    if cfg == 5:
        N = p["N"]
        order = max(0, (N - 1).bit_length())
        idx = np.arange(N)
        hpad = Partial(Hadamard(order), idx, idx)
        return Product(Diag(p["d1"]), Fourier(N), Diag(p["d2"]), Sum(hpad, LowRank(p["U"], p["V"])))
    raise ValueError(cfg)


def c3_flops_per_direction(ncols: int) -> float:
    """~0.56 M FP32 flops per column of C3 with real-pair
    packing — two length-8192 complex FFTs (5 L log2 L each) and the spectrum
    multiply (6 L) per packed column pair."""
    L = 8192
    per_pair = 2 * 5 * L * 13 + 6 * L
    return (ncols / 2) * per_pair


def c5_flops_per_direction(ncols: int, n: int | None = None) -> float:
    """~1.02 G FP64 flops per column of C5 — the length-M
    Bluestein FFT and inverse FFT (5 M log2 M each), the spectrum and chirp /
    diagonal multiplies (6 flops per complex product), the two rank-32 halves
    (8 n r each) and the padded FWHT (2 P log2 P)."""
    N = C5_N if n is None else n
    M = 1 << (2 * N - 1).bit_length()
    P = 1 << max(0, (N - 1).bit_length())
    lm, lp = M.bit_length() - 1, P.bit_length() - 1
    per_col = 2 * 5 * M * lm + 6 * M + 2 * 6 * N + 2 * 8 * N * 32 + 2 * P * lp
    return float(ncols) * per_col


def algorithmic_bytes(cfg: int, ncols: int, n: int | None = None) -> int:
    """Bytes of the minimal number of HBM passes per direction."""
    if cfg == 1:
        N = 1024 if n is None else n
        return 2 * N * ncols * 8
    if cfg == 2:
        N = (1 << 20) if n is None else n
        # 3 passes of read+write of the (N, K) c64 block + the c64 spectrum once
        return 3 * 2 * N * ncols * 8 + N * 8
    if cfg == 3:
        N = 3000 if n is None else n
        return 2 * N * ncols * 4
    if cfg == 4:
        N = 1 << 21 if n is None else 64 * 128 * n
        return 2 * 2 * N * ncols * 8
    if cfg == 5:
        N = C5_N if n is None else n
        M = 1 << (2 * N - 1).bit_length()
        P = 1 << max(0, (N - 1).bit_length())
        e = 16
        p1 = N * ncols * e + N * 32 * e + P * ncols * e
        p2 = P * ncols * e + N * 32 * e + 2 * N * e + M * ncols * e
        p3 = 2 * M * ncols * e + M * e
        p4 = M * ncols * e + 2 * N * e + N * ncols * e
        return p1 + p2 + p3 + p4
    raise ValueError(cfg)
