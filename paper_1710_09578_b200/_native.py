"""ctypes binding of libsmat.so (the C ABI in include/smat.h).

Only the operator classes use this module: they serialise their tree into an
array of ``smat_node`` (one per operator, children by index), build an
immutable device plan once per (dtype, device) and then make one
``smat_apply`` (device tensors) or ``smat_apply_host`` (numpy / CPU tensors)
call per application.  There is deliberately no CPU fallback: if the library
or a CUDA device is missing, every transform raises.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import numpy as np

from .errors import (
    DimensionMismatch,
    LinOpError,
    NotPowerOfTwo,
)

LIB_PATH = Path(__file__).resolve().parent / "libsmat.so"
ABI_VERSION = 3  # SMAT_ABI_VERSION of include/smat.h

# smat_dtype
F32, F64, C64, C128, I32, I64 = range(6)
# smat_kind
(IDENTITY, ZERO, DIAGONAL, DENSE, HADAMARD, FOURIER, CIRCULANT, TOEPLITZ, LOWRANK,
 PRODUCT, SUM, KRON, PARTIAL, ADJOINT, BLOCKDIAG, BLOCKS, SCALED, SPARSE, POLYNOMIAL) = range(19)
CG_STATE = 8  # SMAT_CG_STATE

DTYPE_CODE = {
    np.dtype(np.float32): F32,
    np.dtype(np.float64): F64,
    np.dtype(np.complex64): C64,
    np.dtype(np.complex128): C128,
    np.dtype(np.int32): I32,
    np.dtype(np.int64): I64,
}
CODE_DTYPE = {v: k for k, v in DTYPE_CODE.items()}
REAL_OF = {C64: F32, C128: F64}

# smat_layout
ROW_MAJOR, COL_MAJOR = 0, 1
# status codes
OK, BAD_SHAPE, NOT_POW2, BAD_DTYPE, CUDA_ERROR, BAD_ARG, UNSUPPORTED, OOM = range(8)


class SmatParam(ctypes.Structure):
    _fields_ = [
        ("data", ctypes.c_void_p),
        ("len", ctypes.c_int64),
        ("dtype", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
    ]


class SmatNode(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("n_children", ctypes.c_int32),
        ("first_child", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("iparam", ctypes.c_int64 * 4),
        ("dparam", ctypes.c_double * 2),
        ("param", SmatParam * 4),
    ]


class NativeError(LinOpError, RuntimeError):
    """A failure reported by libsmat.so (CUDA error, unsupported size, ...)."""


_lib = None
_lib_lock = threading.Lock()

_SIGNATURES = {
    "smat_abi_version": ([], ctypes.c_int),
    "smat_last_error": ([], ctypes.c_char_p),
    "smat_plan_build": (
        [ctypes.POINTER(SmatNode), ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
         ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)],
        ctypes.c_int,
    ),
    "smat_probe_peak": ([ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "smat_workspace_bytes": (
        [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
         ctypes.POINTER(ctypes.c_size_t)],
        ctypes.c_int,
    ),
    "smat_apply": (
        [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p,
         ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
        ctypes.c_int,
    ),
    "smat_apply_host": (
        [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p,
         ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32],
        ctypes.c_int,
    ),
    "smat_apply_profiled": (
        [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
         ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float), ctypes.c_int32,
         ctypes.POINTER(ctypes.c_int32), ctypes.c_char_p, ctypes.c_size_t],
        ctypes.c_int,
    ),
    "smat_plan_launches": (
        [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)],
        ctypes.c_int,
    ),
    "smat_plan_describe": ([ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t], ctypes.c_int),
    "smat_plan_shape": (
        [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
         ctypes.POINTER(ctypes.c_int32)],
        ctypes.c_int,
    ),
    "smat_plan_free": ([ctypes.c_void_p], None),
    # device-resident solver steps (solvers.cu)
    "smat_solver_scratch_bytes": ([ctypes.c_int64, ctypes.c_int64], ctypes.c_size_t),
    "smat_cg_init": (
        [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
        ctypes.c_int,
    ),
    "smat_cg_step": (
        [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
        ctypes.c_int,
    ),
    "smat_ista_residual": (
        [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
        ctypes.c_int,
    ),
    "smat_ista_update": (
        [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
        ctypes.c_int,
    ),
    "smat_power_step": (
        [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
         ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
        ctypes.c_int,
    ),
    "smat_soft_threshold": (
        [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p],
        ctypes.c_int,
    ),
    "smat_abs_argmax": (
        [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_size_t, ctypes.c_void_p],
        ctypes.c_int,
    ),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)


def load_library(path: str | Path | None = None):
    """Load libsmat.so (built in-tree by ``paper_1710_09578_b200.build``)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise NativeError(
                f"{p} is missing: build it with `python -m paper_1710_09578_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(str(p))
        for name, (argtypes, restype) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = restype
        if lib.smat_abi_version() != ABI_VERSION:
            raise NativeError(f"{p} has ABI version {lib.smat_abi_version()}, this package needs {ABI_VERSION}: "
                              "rebuild it with `python -m paper_1710_09578_b200.build`")
        if path is None:
            _lib = lib
        return lib


def check(status: int, what: str = "libsmat") -> None:
    if status == OK:
        return
    msg = load_library().smat_last_error().decode(errors="replace")
    if status == BAD_SHAPE:
        raise DimensionMismatch(f"{what}: {msg}")
    if status == NOT_POW2:
        raise NotPowerOfTwo(f"{what}: {msg}")
    if status == BAD_DTYPE:
        raise TypeError(f"{what}: {msg}")
    if status == BAD_ARG:
        raise ValueError(f"{what}: {msg}")
    if status == OOM:
        raise MemoryError(f"{what}: {msg}")
    raise NativeError(f"{what}: status {status}: {msg}")


# ------------------------------------------------------------ serialiser ----
class Serializer:
    """Flattens an operator tree into smat_node records (children by index).

    A Python object that occurs several times in the tree (e.g. a shared
    block of a Blocks grid) is emitted once; the plan compiler builds it once.
    """

    def __init__(self):
        self.records: list[dict] = []
        self.children: list[int] = []
        self.keep: list[np.ndarray] = []
        self.memo: dict[int, int] = {}

    def param(self, arr: np.ndarray | None):
        if arr is None:
            return (0, 0, F64)
        a = np.ascontiguousarray(arr)
        if a.dtype not in DTYPE_CODE:
            if np.issubdtype(a.dtype, np.complexfloating):
                a = a.astype(np.complex128)
            elif np.issubdtype(a.dtype, np.integer):
                a = a.astype(np.int64)
            else:
                a = a.astype(np.float64)
        self.keep.append(a)
        return (a.ctypes.data, a.size, DTYPE_CODE[a.dtype])

    def emit(self, op) -> int:
        key = id(op)
        if key in self.memo:
            return self.memo[key]
        rec = op._smat_record(self)  # dict(kind, rows, cols, iparam, dparam, params, children)
        kids = rec.pop("children", ())
        kid_idx = [self.emit(k) for k in kids]
        first = len(self.children)
        self.children.extend(kid_idx)
        rec["first_child"] = first if kid_idx else 0
        rec["n_children"] = len(kid_idx)
        idx = len(self.records)
        self.records.append(rec)
        self.memo[key] = idx
        return idx

    def arrays(self):
        n = len(self.records)
        nodes = (SmatNode * n)()
        for i, r in enumerate(self.records):
            nd = nodes[i]
            nd.kind = r["kind"]
            nd.n_children = r["n_children"]
            nd.first_child = r["first_child"]
            nd.rows = int(r["rows"])
            nd.cols = int(r["cols"])
            for k, v in enumerate(r.get("iparam", ())):
                nd.iparam[k] = int(v)
            for k, v in enumerate(r.get("dparam", ())):
                nd.dparam[k] = float(v)
            for k, p in enumerate(r.get("params", ())):
                data, length, dt = self.param(p) if not isinstance(p, tuple) else p
                nd.param[k].data = data
                nd.param[k].len = length
                nd.param[k].dtype = dt
        kids = (ctypes.c_int32 * max(1, len(self.children)))(*self.children)
        return nodes, kids


class Plan:
    """An immutable compiled device plan (one per operator tree, dtype, device)."""

    def __init__(self, op, dtype_code: int, device: int):
        lib = load_library()
        ser = Serializer()
        root = ser.emit(op)
        nodes, kids = ser.arrays()
        handle = ctypes.c_void_p()
        check(
            lib.smat_plan_build(nodes, len(ser.records), kids, len(ser.children), root, dtype_code, device,
                                ctypes.byref(handle)),
            f"plan build for {op!r}",
        )
        self._lib = lib
        self.handle = handle
        self.dtype_code = dtype_code
        self.device = device
        self.rows = op.rows
        self.cols = op.cols
        self._ws_cache: dict = {}
        self._ws_bytes: dict = {}
        self._ws_lock = threading.Lock()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and h.value and self._lib is not None:
            try:
                self._lib.smat_plan_free(h)
            except Exception:
                pass
            self.handle = None

    def workspace_bytes(self, direction: int, ncols: int, ldx: int = 0, ldy: int = 0,
                        layout: int = ROW_MAJOR) -> int:
        key = (direction, ncols, ldx, ldy, layout)
        got = self._ws_bytes.get(key)
        if got is None:
            out = ctypes.c_size_t()
            check(self._lib.smat_workspace_bytes(self.handle, direction, ncols, ldx, ldy, layout, ctypes.byref(out)))
            got = self._ws_bytes[key] = int(out.value)
        return got

    def launches(self, direction: int, ncols: int) -> int:
        out = ctypes.c_int64()
        check(self._lib.smat_plan_launches(self.handle, direction, ncols, ctypes.byref(out)))
        return int(out.value)

    def describe(self) -> str:
        buf = ctypes.create_string_buffer(4096)
        check(self._lib.smat_plan_describe(self.handle, buf, 4096))
        return buf.value.decode()

    # -- device path ----------------------------------------------------------
    def workspace(self, direction: int, ncols: int, stream_handle: int | None = None, ldx: int = 0, ldy: int = 0,
                  layout: int = ROW_MAJOR):
        """Cached torch uint8 workspace for (direction, stream) on the plan
        device, grown when a wider block needs more (never one buffer per
        width).  Keyed by stream: applies on one stream are ordered (a buffer
        replaced by a larger one is only reused by later work on the same
        stream), applies on different streams (e.g. from different threads)
        must not share scratch (the reference's concurrent-apply contract,
        core.py:5-7)."""
        import torch

        if stream_handle is None:
            with torch.cuda.device(self.device):
                stream_handle = torch.cuda.current_stream(self.device).cuda_stream
        need = max(1, self.workspace_bytes(direction, ncols, ldx, ldy, layout))
        key = (direction, int(stream_handle))
        ws = self._ws_cache.get(key)
        if ws is not None and ws.numel() >= need:
            return ws
        with self._ws_lock:
            ws = self._ws_cache.get(key)
            if ws is None or ws.numel() < need:
                ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{self.device}")
                self._ws_cache[key] = ws
        return ws

    def apply_device(self, direction: int, x, x_code: int, y, ncols: int, stream_handle: int, ldx: int = 0,
                     ldy: int = 0, layout: int = ROW_MAJOR) -> None:
        ws = self.workspace(direction, ncols, stream_handle, ldx, ldy, layout)
        check(
            self._lib.smat_apply(self.handle, direction, ctypes.c_void_p(x.data_ptr()), x_code, ldx,
                                 ctypes.c_void_p(y.data_ptr()), ldy, ncols, layout, ctypes.c_void_p(ws.data_ptr()),
                                 ws.numel(), ctypes.c_void_p(stream_handle)),
            "smat_apply",
        )

    def apply_profiled(self, direction: int, x, x_code: int, y, ncols: int, stream_handle: int):
        """One smat_apply with per-launch CUDA events: [(label, ms), ...]."""
        ws = self.workspace(direction, ncols, stream_handle)
        cap = 256
        ms = (ctypes.c_float * cap)()
        n = ctypes.c_int32()
        labels = ctypes.create_string_buffer(cap * 32)
        check(
            self._lib.smat_apply_profiled(self.handle, direction, ctypes.c_void_p(x.data_ptr()), x_code,
                                          ctypes.c_void_p(y.data_ptr()), ncols, ctypes.c_void_p(ws.data_ptr()),
                                          ws.numel(), ctypes.c_void_p(stream_handle), ms, cap,
                                          ctypes.byref(n), labels, len(labels)),
            "smat_apply_profiled",
        )
        names = labels.value.decode().split("\n")
        return [(names[i], float(ms[i])) for i in range(n.value)]

    # -- host path --------------------------------------------------------------
    def apply_host(self, direction: int, x_ptr: int, x_code: int, y_ptr: int, ncols: int,
                   chunk_cols: int = 0, ldx: int = 0, ldy: int = 0, layout: int = ROW_MAJOR) -> None:
        check(
            self._lib.smat_apply_host(self.handle, direction, ctypes.c_void_p(x_ptr), x_code, ldx,
                                      ctypes.c_void_p(y_ptr), ldy, ncols, layout, chunk_cols),
            "smat_apply_host",
        )


def probe_peak(kind: int, device: int = 0) -> float:
    """Measured arithmetic peak in TFLOP/s (smat_probe_peak): 0 DFMA, 1 DMMA,
    2 DFMA + DMMA side by side, 3 FFMA2."""
    out = ctypes.c_double()
    check(load_library().smat_probe_peak(kind, device, ctypes.byref(out)), "smat_probe_peak")
    return float(out.value)
