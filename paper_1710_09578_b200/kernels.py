"""Kernel-level transform API (reference: pkg/src/linopkit/kernels.py:39-223).

``dft``, ``fwht``, ``circular_convolve`` and ``DftPlan``/``get_plan`` keep the
reference names, argument meaning and errors, but every transform runs on the
device through a single-leaf plan of libsmat.so (Fourier / Hadamard /
Circulant).  DFT conventions (kernels.py:4-7): forward X_j = sum_k x_k w^(jk),
w = exp(-2i pi / n); the inverse divides by n.
"""

from __future__ import annotations

import functools

import numpy as np

from .core import _is_torch
from .errors import DimensionMismatch, EmptyInput, NotPowerOfTwo


def is_power_of_two(n):
    return n >= 1 and (n & (n - 1)) == 0


def next_power_of_two(n):
    m = 1
    while m < n:
        m <<= 1
    return m


def _rows(x):
    return x.shape[0] if (_is_torch(x) or hasattr(x, "shape")) else np.asarray(x).shape[0]


class DftPlan:
    """Length-n DFT plan (kernels.py:59-147): radix/four-step FFT for powers of
    two, Bluestein chirp-z otherwise; tables live on the device."""

    def __init__(self, n):
        n = int(n)
        if n < 1:
            raise EmptyInput("DFT length must be >= 1")
        self.n = n
        from .leaves import Fourier

        self._op = Fourier(n)
        self._inv = None

    def execute(self, x, inverse=False):
        """Transform along axis 0; ``x`` is ``(n,)`` or ``(n, k)`` (kernels.py:127-147)."""
        rows = _rows(x)
        if rows != self.n:
            raise DimensionMismatch(f"plan length {self.n}, input has {rows} rows")
        if not inverse:
            return self._op.forward(x)
        if self._inv is None:
            from .composites import Scaled

            self._inv = Scaled(self._op.adjoint(), 1.0 / self.n)  # IDFT = F^H / n
        return self._inv.forward(x)


@functools.lru_cache(maxsize=64)
def get_plan(n):
    """Shared plan cache (kernels.py:150-153)."""
    return DftPlan(n)


def dft(x, inverse=False):
    """Unnormalized DFT of ``x`` along axis 0 (inverse includes the 1/n)."""
    arr = x if _is_torch(x) else np.asarray(x)
    if arr.shape[0] == 0:
        raise EmptyInput("cannot transform an empty vector")
    return get_plan(arr.shape[0]).execute(arr, inverse=inverse)


@functools.lru_cache(maxsize=64)
def _hadamard(order):
    from .leaves import Hadamard

    return Hadamard(order)


def fwht(x):
    """Walsh-Hadamard transform H_n @ x, Sylvester order (kernels.py:164-190).

    Stage order stride-1-first like the reference, so float64 results are
    bit-identical to it; int32/int64 inputs stay exact integers."""
    arr = x if _is_torch(x) else np.asarray(x)
    n = arr.shape[0]
    if not is_power_of_two(n):
        raise NotPowerOfTwo(f"Walsh-Hadamard length must be a power of two, got {n}")
    return _hadamard(n.bit_length() - 1).forward(arr)


def circular_convolve(c, x):
    """Circular convolution y_i = sum_k c_((i-k) mod n) x_k (kernels.py:193-223);
    real inputs give a real result."""
    carr = np.asarray(c)
    xarr = x if _is_torch(x) else np.asarray(x)
    if carr.ndim != 1:
        raise ValueError("convolution kernel must be 1-D")
    if carr.shape[0] == 0:
        raise EmptyInput("convolution kernel must be nonempty")
    if xarr.shape[0] != carr.shape[0]:
        raise DimensionMismatch(f"kernel length {carr.shape[0]} != input rows {xarr.shape[0]}")
    from .leaves import Circulant

    return Circulant(carr).forward(xarr)
