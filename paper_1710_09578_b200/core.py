"""Operator interface: validation, scalar fields, dense oracle, adjoint, footprint.

Mirrors the reference contract of ``LinearOperator`` (pkg/src/linopkit/core.py:76-226):
public ``forward``/``backward`` validate shape and dtype exactly like the
reference (core.py:128-167, same exception classes and messages) and then hand
the whole operator tree to the native engine: the tree is compiled once per
(working dtype, device) into a device plan (libsmat.so, include/smat.h) and
each application is ONE native call.  There is no CPU fallback.

Deliberate, documented deviation from the reference: the
reference up-casts every input to float64/complex128 (core.py:63-73).  Here the
working precision follows the input — float32/complex64 inputs are computed in
single precision, float64/complex128 (and integers, as in the reference) in
double precision — and integer inputs to pure Walsh-Hadamard trees stay exact
integers (int32 in, int32 out).  The scalar *field* (real vs complex) follows
the reference's promotion lattice (core.py:34-38).

Accepted inputs: anything ``numpy.asarray`` accepts (computed through the
pipelined host entry point ``smat_apply_host``; the result is a numpy array),
CPU torch tensors (result on the CPU) and CUDA torch tensors (result on the
same device, computed on the current stream with ``smat_apply``).
"""

from __future__ import annotations

import enum
import threading

import numpy as np

from . import _native
from .errors import DimensionMismatch, MaterializationTooLarge

DEFAULT_DENSE_CAP_BYTES = 2 ** 31  # 2 GiB materialization guard (core.py:16)

# Host blocks of at least this many bytes are streamed through the device in
# column chunks: H2D copies, device passes and D2H copies of different chunks
# overlap on three streams.  A column chunk of a row-major block is a pitched
# copy; the box copies 512- and 256-byte rows at the full link rate (~55 GB/s
# one way, ~64-69 GB/s with H2D and D2H overlapped) but 64-byte rows at half
# (tools/pcie2d_probe.py), so chunks are the widest of 512 / 256 / 128-byte
# rows that still give two or more chunks.  Measured e2e gains: C2 3.2k ->
# 4.1k, C4 1.59k -> 1.76k, C5 1.49k -> 2.34k columns/s.  Smaller blocks move as
# one contiguous DMA each way.
HOST_CHUNK_BYTES = 256 << 20


def _host_chunk(ncols: int, n_in: int, n_out: int, esz: int) -> int:
    """Columns per host-path chunk (0 = one contiguous DMA each way)."""
    if max(n_in, n_out) * ncols * esz < HOST_CHUNK_BYTES:
        return 0
    for row_bytes in (512, 256, 128):
        c = max(1, row_bytes // esz)
        if ncols >= 2 * c:
            return c
    return 0


class ScalarField(enum.Enum):
    """Scalar field of an operator or batch: real or complex (core.py:19-31)."""

    REAL64 = "real64"
    COMPLEX128 = "complex128"

    @property
    def dtype(self):
        return np.complex128 if self is ScalarField.COMPLEX128 else np.float64

    @property
    def size_bytes(self):
        return 16 if self is ScalarField.COMPLEX128 else 8


def promote_field(a, b):
    """Complex wins (core.py:34-38)."""
    if a is ScalarField.COMPLEX128 or b is ScalarField.COMPLEX128:
        return ScalarField.COMPLEX128
    return ScalarField.REAL64


def as_field(value):
    """Coerce a ScalarField, dtype or string into a ScalarField (core.py:41-55)."""
    if isinstance(value, ScalarField):
        return value
    if isinstance(value, str):
        try:
            return ScalarField(value.lower())
        except ValueError:
            raise ValueError(f"unknown scalar field {value!r}") from None
    dt = np.dtype(value)
    if np.issubdtype(dt, np.complexfloating):
        return ScalarField.COMPLEX128
    if np.issubdtype(dt, np.number) or np.issubdtype(dt, np.bool_):
        return ScalarField.REAL64
    raise TypeError(f"no scalar field for dtype {dt}")


def field_of(arr):
    """ScalarField of an array (complex dtypes map to COMPLEX128)."""
    return as_field(_np_dtype(arr))


# --------------------------------------------------------------- dtypes -----
_SINGLE = {np.dtype(np.float32), np.dtype(np.complex64), np.dtype(np.float16)}


def _is_torch(x) -> bool:
    t = type(x)
    return t.__module__.startswith("torch") and t.__name__ in ("Tensor", "Parameter")


_TORCH_NP: dict = {}


def _np_dtype(x):
    if _is_torch(x):
        dt = _TORCH_NP.get(x.dtype)
        if dt is None:
            import torch

            dt = np.dtype(torch.empty((), dtype=x.dtype).numpy().dtype) if x.dtype != torch.bfloat16 \
                else np.dtype(np.float32)
            _TORCH_NP[x.dtype] = dt
        return dt
    return np.asarray(x).dtype if not hasattr(x, "dtype") else np.dtype(x.dtype)


def coerce_array(x, name="x"):
    """Validate a numeric 1-D/2-D input (core.py:63-73) WITHOUT up-casting.

    Returns a numpy array; raises TypeError for non-numeric input and
    ValueError for ndim not in (1, 2), as the reference does.
    """
    arr = np.asarray(x)
    if arr.dtype == object or not (
        np.issubdtype(arr.dtype, np.number) or np.issubdtype(arr.dtype, np.bool_)
    ):
        raise TypeError(f"{name} must be numeric, got dtype {arr.dtype}")
    if arr.ndim not in (1, 2):
        raise ValueError(f"{name} must be 1-D or 2-D, got ndim {arr.ndim}")
    return arr


def _work_codes(op, xdt: np.dtype):
    """(plan dtype code, input dtype code) for an input of numpy dtype xdt
    (memoised per operator and dtype: the tree is immutable)."""
    memo = op.__dict__.setdefault("_codes_memo", {})
    got = memo.get(xdt)
    if got is None:
        got = memo[xdt] = _work_codes_uncached(op, xdt)
    return got


def _work_codes_uncached(op, xdt: np.dtype):
    if (np.issubdtype(xdt, np.integer) and op._int_exact()
            and xdt in (np.dtype(np.int32), np.dtype(np.int64))):
        code = _native.DTYPE_CODE[xdt]
        return code, code
    single = xdt in _SINGLE
    x_cplx = np.issubdtype(xdt, np.complexfloating)
    out_field = promote_field(op.field, ScalarField.COMPLEX128 if x_cplx else ScalarField.REAL64)
    if out_field is ScalarField.COMPLEX128:
        plan = _native.C64 if single else _native.C128
        xcode = plan if x_cplx else _native.REAL_OF[plan]
    else:
        plan = _native.F32 if single else _native.F64
        xcode = plan
    return plan, xcode


_TORCH_OF_CODE: dict = {}


def _torch_dtype(code):
    if not _TORCH_OF_CODE:
        import torch

        _TORCH_OF_CODE.update({
            _native.F32: torch.float32, _native.F64: torch.float64, _native.C64: torch.complex64,
            _native.C128: torch.complex128, _native.I32: torch.int32, _native.I64: torch.int64,
        })
    return _TORCH_OF_CODE[code]


def _raw_stream(torch, dev: int) -> int:
    """The current CUDA stream handle of `dev` (torch's raw accessor when
    present: the public current_stream() costs several microseconds)."""
    fn = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    return fn(dev) if fn is not None else torch.cuda.current_stream(dev).cuda_stream


def _block_layout(s0: int, s1: int, rows: int, ncols: int):
    """(leading dimension, smat layout) of a 2-D block with element strides
    (s0, s1), or (-1, ROW_MAJOR) when it needs a dense copy first.  Dense
    row-major blocks report ld 0."""
    if ncols == 1 or s1 == 1:
        ld = s0 if rows > 1 else ncols
        if ld == ncols:
            return 0, _native.ROW_MAJOR
        if ld > ncols:
            return ld, _native.ROW_MAJOR
    if s0 == 1 and s1 >= rows:
        return s1, _native.COL_MAJOR
    return -1, _native.ROW_MAJOR


def _default_device() -> int:
    import torch

    if not torch.cuda.is_available():
        raise _native.NativeError(
            "no CUDA device is visible: the structured transforms run only on the GPU "
            "(libsmat.so, sm_100a); there is no CPU fallback"
        )
    return torch.cuda.current_device()


class LinearOperator:
    """Abstract matrix-free operator A with validated forward x -> A x and
    backward y -> A^H y (core.py:76-226).

    Subclasses call ``_init_shape`` and implement ``_smat_record`` (their
    node in the serialised tree handed to the native plan compiler),
    ``_param_bytes`` and optionally ``_children``.
    """

    _shape = None
    _field = ScalarField.REAL64

    def _init_shape(self, rows, cols, field):
        rows = int(rows)
        cols = int(cols)
        if rows < 1 or cols < 1:
            raise ValueError(f"operator shape must be positive, got ({rows}, {cols})")
        self._shape = (rows, cols)
        self._field = field

    @property
    def shape(self):
        return self._shape

    @property
    def rows(self):
        return self._shape[0]

    @property
    def cols(self):
        return self._shape[1]

    # fastmat-style aliases (paper API: numN x numM)
    @property
    def numN(self):
        return self._shape[0]

    @property
    def numM(self):
        return self._shape[1]

    @property
    def field(self):
        return self._field

    # -- hooks supplied by subclasses -----------------------------------------
    def _smat_record(self, ser):
        raise NotImplementedError

    def _param_bytes(self):
        raise NotImplementedError

    def _children(self):
        return ()

    def _int_exact(self) -> bool:
        """True when integer inputs can stay exact integers (pure ±1 sums)."""
        return False

    # -- native plans -----------------------------------------------------------
    def _plan(self, code: int, device: int):
        plan = self.__dict__.get("_plans", {}).get((code, device))
        if plan is not None:  # (plans are never replaced once built)
            return plan
        lock = self.__dict__.setdefault("_plan_lock", threading.Lock())
        with lock:
            cache = self.__dict__.setdefault("_plans", {})
            plan = cache.get((code, device))
            if plan is None:
                plan = _native.Plan(self, code, device)
                cache[(code, device)] = plan
            return plan

    def plan_for(self, dtype, device: int | None = None):
        """The compiled device plan used for inputs of numpy dtype ``dtype``."""
        code, _ = _work_codes(self, np.dtype(dtype))
        return self._plan(code, _default_device() if device is None else device)

    # -- validated public entry points ------------------------------------------
    def forward(self, x):
        """Apply the operator: returns A @ x (core.py:128-149)."""
        return self._apply(x, 0, "x")

    def backward(self, y):
        """Apply the Hermitian adjoint: returns A^H @ y (core.py:151-167)."""
        return self._apply(y, 1, "y")

    def __matmul__(self, x):
        if isinstance(x, LinearOperator):
            from .composites import Product

            return Product(self, x)
        return self.forward(x)

    def __add__(self, other):
        if not isinstance(other, LinearOperator):
            return NotImplemented
        from .composites import Sum

        return Sum(self, other)

    def __mul__(self, other):
        if not isinstance(other, LinearOperator):
            return NotImplemented
        from .composites import Product

        return Product(self, other)

    def _mismatch(self, direction, got, shape_in):
        if direction == 0:
            return DimensionMismatch(
                f"{self!r} expects input with {self.cols} rows, got {got} "
                f"(operator shape {self.shape}, input shape {shape_in})"
            )
        return DimensionMismatch(
            f"adjoint of {self!r} expects input with {self.rows} rows, got "
            f"{got} (operator shape {self.shape}, input shape {shape_in})"
        )

    def _apply(self, x, direction, name):
        n_in = self.cols if direction == 0 else self.rows
        n_out = self.rows if direction == 0 else self.cols
        if _is_torch(x):
            return self._apply_torch(x, direction, name, n_in, n_out)
        arr = coerce_array(x, name)
        squeeze = arr.ndim == 1
        a2 = arr[:, None] if squeeze else arr
        if a2.shape[0] != n_in:
            raise self._mismatch(direction, a2.shape[0], arr.shape[:1] if squeeze else arr.shape)
        pcode, xcode = _work_codes(self, a2.dtype)
        ncols = a2.shape[1]
        out = np.empty((n_out, ncols), dtype=_native.CODE_DTYPE[pcode])
        if ncols:
            xin = a2 if a2.dtype == _native.CODE_DTYPE[xcode] else a2.astype(_native.CODE_DTYPE[xcode])
            ld, layout = _block_layout(xin.strides[0] // xin.itemsize if xin.strides[0] % xin.itemsize == 0 else -1,
                                       xin.strides[1] // xin.itemsize if xin.strides[1] % xin.itemsize == 0 else -1,
                                       n_in, ncols)
            if ld < 0:
                xin = np.ascontiguousarray(xin)
                ld, layout = 0, _native.ROW_MAJOR
            if layout == _native.COL_MAJOR:  # the result keeps the input's (Fortran) layout
                out = np.empty((n_out, ncols), dtype=out.dtype, order="F")
            plan = self._plan(pcode, _default_device())
            esz = max(xin.itemsize, out.itemsize)
            plan.apply_host(direction, xin.ctypes.data, xcode, out.ctypes.data, ncols,
                            _host_chunk(ncols, n_in, n_out, esz) if layout == _native.ROW_MAJOR else 0,
                            ldx=ld, layout=layout)
        return out[:, 0] if squeeze else out

    def _apply_torch(self, x, direction, name, n_in, n_out):
        import torch

        ints = (torch.int8, torch.uint8, torch.int16, torch.int32, torch.int64)
        if not (x.dtype.is_floating_point or x.dtype.is_complex or x.dtype == torch.bool or x.dtype in ints):
            raise TypeError(f"{name} must be numeric, got dtype {x.dtype}")
        if x.dim() not in (1, 2):
            raise ValueError(f"{name} must be 1-D or 2-D, got ndim {x.dim()}")
        squeeze = x.dim() == 1
        x2 = x[:, None] if squeeze else x
        if x2.shape[0] != n_in:
            raise self._mismatch(direction, x2.shape[0], tuple(x.shape[:1]) if squeeze else tuple(x.shape))
        xdt = _np_dtype(x2)
        pcode, xcode = _work_codes(self, xdt)
        ncols = x2.shape[1]
        xdt_t = _torch_dtype(xcode)
        # strided views (column slices of a wider block, transposes) are
        # handed to the engine with their leading dimension: no copy here
        xin = x2 if x2.dtype == xdt_t else x2.to(xdt_t)
        ld, layout = _block_layout(xin.stride(0), xin.stride(1), n_in, ncols)
        if ld < 0:
            xin = xin.contiguous()
            ld, layout = 0, _native.ROW_MAJOR
        def _out(**kw):
            # the result keeps the input's layout (column-major in, column-major out)
            if layout == _native.COL_MAJOR:
                return torch.empty((ncols, n_out), dtype=_torch_dtype(pcode), **kw).t()
            return torch.empty((n_out, ncols), dtype=_torch_dtype(pcode), **kw)

        if not x2.is_cuda:
            # host tensor: pinned (or pageable) memory through the pipelined host path
            out = _out(pin_memory=xin.is_pinned())
            if ncols:
                plan = self._plan(pcode, _default_device())
                esz = max(xin.element_size(), out.element_size())
                plan.apply_host(direction, xin.data_ptr(), xcode, out.data_ptr(), ncols,
                                _host_chunk(ncols, n_in, n_out, esz) if layout == _native.ROW_MAJOR else 0,
                                ldx=ld, layout=layout)
            return out[:, 0] if squeeze else out
        cur = torch.cuda.current_device()
        dev = x2.device.index if x2.device.index is not None else cur
        out = _out(device=x2.device)
        if ncols:
            plan = self._plan(pcode, dev)
            if dev == cur:
                plan.apply_device(direction, xin, xcode, out, ncols, _raw_stream(torch, dev), ldx=ld, layout=layout)
            else:
                with torch.cuda.device(dev):
                    stream = torch.cuda.current_stream(dev)
                    plan.apply_device(direction, xin, xcode, out, ncols, stream.cuda_stream, ldx=ld, layout=layout)
        return out[:, 0] if squeeze else out

    # -- derived operations --------------------------------------------------------
    def adjoint(self):
        """The Hermitian adjoint as an operator (wraps, does not copy)."""
        return Adjoint(self)

    @property
    def H(self):
        return self.adjoint()

    def to_dense(self, cap_bytes=DEFAULT_DENSE_CAP_BYTES):
        """Materialize the dense matrix; column j is forward(e_j) (core.py:182-204)."""
        n, m = self.shape
        need = n * m * self.field.size_bytes
        if need >= cap_bytes:
            raise MaterializationTooLarge(
                f"dense {n}x{m} {self.field.value} needs {need} bytes "
                f"(cap {cap_bytes})"
            )
        out = np.empty((n, m), dtype=self.field.dtype)
        block = max(1, min(m, (1 << 26) // max(1, n * self.field.size_bytes)))
        for j0 in range(0, m, block):
            j1 = min(m, j0 + block)
            basis = np.zeros((m, j1 - j0), dtype=self.field.dtype)
            basis[np.arange(j0, j1), np.arange(j1 - j0)] = 1
            out[:, j0:j1] = self.forward(basis)
        return out

    def footprint_bytes(self):
        """Host parameter bytes of the tree, each instance once (core.py:206-223)."""
        seen = set()
        total = 0
        stack = [self]
        while stack:
            op = stack.pop()
            if id(op) in seen:
                continue
            seen.add(id(op))
            total += op._param_bytes()
            stack.extend(op._children())
        return total

    def __repr__(self):
        return f"{type(self).__name__}(shape={self.shape}, field={self.field.value})"


class Adjoint(LinearOperator):
    """Hermitian-adjoint view of a base operator (core.py:229-253)."""

    def __init__(self, base):
        self.base = base
        self._init_shape(base.cols, base.rows, base.field)

    def adjoint(self):
        return self.base

    def _int_exact(self):
        return self.base._int_exact()

    def _smat_record(self, ser):
        return dict(kind=_native.ADJOINT, rows=self.rows, cols=self.cols, children=(self.base,))

    def _param_bytes(self):
        return 8

    def _children(self):
        return (self.base,)

    def __repr__(self):
        return f"Adjoint({self.base!r})"
