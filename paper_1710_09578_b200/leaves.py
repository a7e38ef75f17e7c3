"""Concrete structured operators (reference: pkg/src/linopkit/leaves.py).

Each class keeps the reference constructor signature, validation and error
classes, and stores only its defining parameters on the host (the dense
footprint accounting of core.py:206-223).  Spectra, chirps and twiddles are
computed ON THE DEVICE in fp64 when the operator's plan is compiled
(libsmat.so), then stored at the working precision.

Paper/fastmat aliases: ``Diag`` = ``Diagonal``, ``Matrix`` = ``Dense``.
``LowRank`` (U·diag(s)·V^H) is new: the reference expresses it as
``Product(Dense(U), Dense(V^H))``.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .core import LinearOperator, ScalarField, as_field, field_of, promote_field
from .errors import EmptyInput, IndexOutOfRange, OrderTooLarge

MAX_HADAMARD_ORDER = 30  # leaves.py:16


def _next_pow2(n: int) -> int:
    m = 1
    while m < n:
        m <<= 1
    return m


def _as_param_vector(d, name):
    """1-D nonempty parameter, stored as float64/complex128 (leaves.py:19-25)."""
    arr = np.asarray(d)
    if arr.ndim != 1:
        raise ValueError(f"{name} must be 1-D, got ndim {arr.ndim}")
    if arr.shape[0] == 0:
        raise EmptyInput(f"{name} must be nonempty")
    return arr.astype(as_field(arr.dtype).dtype, copy=False)


class Dense(LinearOperator):
    """Unstructured operator over explicitly stored entries (leaves.py:28-49)."""

    def __init__(self, entries):
        arr = np.asarray(entries)
        if arr.ndim != 2:
            raise ValueError(f"entries must be 2-D, got ndim {arr.ndim}")
        if arr.size == 0:
            raise EmptyInput("entries must be nonempty")
        self.entries = np.ascontiguousarray(arr, dtype=as_field(arr.dtype).dtype)
        self._init_shape(arr.shape[0], arr.shape[1], field_of(self.entries))

    def _smat_record(self, ser):
        return dict(kind=_native.DENSE, rows=self.rows, cols=self.cols, params=(self.entries,))

    def _param_bytes(self):
        return self.entries.nbytes


Matrix = Dense


class Zero(LinearOperator):
    """All-zeros operator (leaves.py:52-65)."""

    def __init__(self, rows, cols):
        self._init_shape(rows, cols, ScalarField.REAL64)

    def _int_exact(self):
        return True

    def _smat_record(self, ser):
        return dict(kind=_native.ZERO, rows=self.rows, cols=self.cols)

    def _param_bytes(self):
        return 16


class Identity(LinearOperator):
    """Identity (leaves.py:68-79); forward returns a new array."""

    def __init__(self, n):
        self._init_shape(n, n, ScalarField.REAL64)

    def _int_exact(self):
        return True

    def _smat_record(self, ser):
        return dict(kind=_native.IDENTITY, rows=self.rows, cols=self.cols)

    def _param_bytes(self):
        return 8


class Diagonal(LinearOperator):
    """Square operator scaling entry i by d[i] (leaves.py:82-97)."""

    def __init__(self, d):
        self.d = _as_param_vector(d, "diagonal")
        n = self.d.shape[0]
        self._init_shape(n, n, field_of(self.d))

    def _smat_record(self, ser):
        return dict(kind=_native.DIAGONAL, rows=self.rows, cols=self.cols, params=(self.d,))

    def _param_bytes(self):
        return self.d.nbytes


Diag = Diagonal


class Fourier(LinearOperator):
    """Unnormalized DFT matrix, entry (j, k) = w^(jk), w = exp(-2i pi/n)
    (leaves.py:162-178).  Forward is the FFT, backward F^H = n * IDFT; any n
    (Bluestein chirp-z for non powers of two, kernels.py:83-93)."""

    def __init__(self, n):
        self._init_shape(n, n, ScalarField.COMPLEX128)

    def _smat_record(self, ser):
        return dict(kind=_native.FOURIER, rows=self.rows, cols=self.cols)

    def _param_bytes(self):
        return 8


class Hadamard(LinearOperator):
    """Sylvester ±1 matrix of size 2^order (leaves.py:181-204); forward =
    backward = the fast Walsh-Hadamard transform."""

    def __init__(self, order):
        order = int(order)
        if order < 0:
            raise ValueError(f"order must be >= 0, got {order}")
        if order > MAX_HADAMARD_ORDER:
            raise OrderTooLarge(f"order {order} exceeds the {MAX_HADAMARD_ORDER} cap")
        self.order = order
        n = 1 << order
        self._init_shape(n, n, ScalarField.REAL64)

    def _int_exact(self):
        return True

    def _smat_record(self, ser):
        return dict(kind=_native.HADAMARD, rows=self.rows, cols=self.cols, iparam=(self.order,))

    def _param_bytes(self):
        return 8


class Circulant(LinearOperator):
    """Circulant operator defined by its first column c (leaves.py:207-234):
    y = IFFT(FFT(c) * FFT(x)); backward uses conj(FFT(c)).  The spectrum
    multiply is fused between the forward and inverse device transforms."""

    def __init__(self, c):
        self.c = _as_param_vector(c, "first column")
        n = self.c.shape[0]
        self._init_shape(n, n, field_of(self.c))
        self._spectrum = None

    @property
    def spectrum(self):
        """dft(c), computed on the device (cached)."""
        if self._spectrum is None:
            from .kernels import dft

            self._spectrum = dft(self.c.astype(np.complex128))
        return self._spectrum

    def _smat_record(self, ser):
        return dict(kind=_native.CIRCULANT, rows=self.rows, cols=self.cols, params=(self.c,))

    def _param_bytes(self):
        return self.c.nbytes + 16 * self.rows


class Toeplitz(LinearOperator):
    """Toeplitz operator from its first column and the rest of its first row
    (leaves.py:237-290); T[i, j] = col[i-j] (i >= j) else row_rest[j-i-1].
    Applied through a circulant embedding of length next_pow2(n + m - 1)
    with zero-pad on load and truncation on store fused into the FFT passes."""

    def __init__(self, first_col, first_row_rest=()):
        self.first_col = _as_param_vector(first_col, "first column")
        row = np.asarray(first_row_rest)
        if row.ndim != 1:
            raise ValueError("first_row_rest must be 1-D")
        self.first_row_rest = row.astype(as_field(row.dtype).dtype, copy=False) \
            if row.size else np.zeros(0)
        n = self.first_col.shape[0]
        m = self.first_row_rest.shape[0] + 1
        self._embed_len = _next_pow2(n + m - 1)
        field = field_of(self.first_col)
        if self.first_row_rest.size:
            field = promote_field(field, field_of(self.first_row_rest))
        self._init_shape(n, m, field)

    def _smat_record(self, ser):
        return dict(kind=_native.TOEPLITZ, rows=self.rows, cols=self.cols,
                    params=(self.first_col, self.first_row_rest))

    def _param_bytes(self):
        return self.first_col.nbytes + self.first_row_rest.nbytes + 16 * self._embed_len


class LowRank(LinearOperator):
    """Rank-r operator U·diag(s)·V^H with U (n x r), V (m x r), optional s (r).

    New type (no reference class); the reference algebra expresses it as
    Product(Dense(U), [Diagonal(s)], Dense(V^H)).  Forward contracts V^H x
    (split-K reduction) and expands with U; backward V·diag(conj s)·U^H y."""

    def __init__(self, U, V, s=None):
        u = np.asarray(U)
        v = np.asarray(V)
        if u.ndim != 2 or v.ndim != 2:
            raise ValueError("LowRank factors must be 2-D")
        if u.size == 0 or v.size == 0:
            raise EmptyInput("LowRank factors must be nonempty")
        if u.shape[1] != v.shape[1]:
            raise ValueError(f"LowRank rank mismatch: U has {u.shape[1]} columns, V has {v.shape[1]}")
        self.U = np.ascontiguousarray(u, dtype=as_field(u.dtype).dtype)
        self.V = np.ascontiguousarray(v, dtype=as_field(v.dtype).dtype)
        self.rank = u.shape[1]
        field = promote_field(field_of(self.U), field_of(self.V))
        self.s = None
        if s is not None:
            self.s = _as_param_vector(s, "singular values")
            if self.s.shape[0] != self.rank:
                raise ValueError("LowRank s must have one entry per rank")
            field = promote_field(field, field_of(self.s))
        self._init_shape(u.shape[0], v.shape[0], field)

    def _smat_record(self, ser):
        return dict(kind=_native.LOWRANK, rows=self.rows, cols=self.cols, iparam=(self.rank,),
                    params=(self.U, self.V, self.s if self.s is not None else (0, 0, _native.F64)))

    def _param_bytes(self):
        return self.U.nbytes + self.V.nbytes + (self.s.nbytes if self.s is not None else 0)


class Sparse(LinearOperator):
    """Compressed-sparse-row operator built from (row, col, value) triplets
    (leaves.py:100-159).  Duplicate coordinates are summed; the
    conjugate-transposed CSR is built once when the device plan is compiled, so
    the backward transform also runs in O(nnz) (one warp per output row).
    """

    def __init__(self, rows, cols, triplets):
        tri = list(triplets)
        if tri:
            i = np.asarray([t[0] for t in tri], dtype=np.int64)
            j = np.asarray([t[1] for t in tri], dtype=np.int64)
            v = np.asarray([t[2] for t in tri])
        else:
            i = np.zeros(0, dtype=np.int64)
            j = np.zeros(0, dtype=np.int64)
            v = np.zeros(0)
        self._from_arrays(rows, cols, i, j, v)

    def _from_arrays(self, rows, cols, i, j, v):
        """CSR assembly from coordinate arrays (the triplet constructor's body;
        also a bulk path for large operators)."""
        rows = int(rows)
        cols = int(cols)
        i = np.asarray(i, dtype=np.int64)
        j = np.asarray(j, dtype=np.int64)
        v = np.asarray(v)
        if i.size and (i.min() < 0 or i.max() >= rows or j.min() < 0 or j.max() >= cols):
            raise IndexOutOfRange(f"triplet index outside {rows}x{cols} matrix")
        dtype = as_field(v.dtype).dtype if v.size else np.float64
        v = v.astype(dtype)
        # canonical CSR: rows ascending, columns ascending within a row,
        # duplicates summed in triplet order (csr_matrix.sum_duplicates)
        order = np.lexsort((j, i))
        i, j, v = i[order], j[order], v[order]
        if i.size:
            key = i * cols + j
            first = np.concatenate(([True], key[1:] != key[:-1]))
            grp = np.cumsum(first) - 1
            vals = np.zeros(int(first.sum()), dtype=dtype)
            np.add.at(vals, grp, v)
            i, j, v = i[first], j[first], vals
        self._row_ptr = np.zeros(rows + 1, dtype=np.int64)
        np.add.at(self._row_ptr, i + 1, 1)
        self._row_ptr = np.cumsum(self._row_ptr)
        self._col_idx = np.ascontiguousarray(j, dtype=np.int64)
        self._values = np.ascontiguousarray(v, dtype=dtype)
        self._init_shape(rows, cols, field_of(self._values))

    @property
    def row_ptr(self):
        return self._row_ptr

    @property
    def col_idx(self):
        return self._col_idx

    @property
    def values(self):
        return self._values

    @property
    def nnz(self):
        return int(self._values.size)

    def _smat_record(self, ser):
        return dict(kind=_native.SPARSE, rows=self.rows, cols=self.cols,
                    params=(self._row_ptr, self._col_idx, self._values))

    def _param_bytes(self):
        # both CSR copies, with scipy's index width (leaves.py:154-158)
        idx = 4 if max(self.rows, self.cols, self.nnz) < 2**31 else 8
        return 2 * (self._values.nbytes + self.nnz * idx) + (self.rows + 1 + self.cols + 1) * idx


class Parametric(LinearOperator):
    """Operator whose entries come from a function f(i, j) (leaves.py:290-322).

    The reference evaluates f row by row on every application.  Here the
    entries are evaluated once, when the device plan is compiled, into a
    device-resident dense factor (the host keeps only f and the shape); the
    applications are then dense GEMM passes.
    """

    def __init__(self, f, rows, cols, field=ScalarField.COMPLEX128):
        self.f = f
        self._init_shape(rows, cols, as_field(field))

    def _entries(self):
        dt = self.field.dtype
        out = np.empty((self.rows, self.cols), dtype=dt)
        for i in range(self.rows):
            out[i] = np.fromiter((self.f(i, j) for j in range(self.cols)), dtype=dt, count=self.cols)
        return out

    def _smat_record(self, ser):
        return dict(kind=_native.DENSE, rows=self.rows, cols=self.cols, params=(self._entries(),))

    def _param_bytes(self):
        return 24  # function reference plus the two dimensions
