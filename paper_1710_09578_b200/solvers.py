"""Iterative matrix-free algorithms on the device (reference:
pkg/src/linopkit/solvers.py).

Same entry points, options, result types, validation and exceptions as the
reference: ``cg_solve``, ``ista``, ``omp``, ``power_iteration`` and
``soft_threshold``.  The difference is where the iteration lives:

* every iterate, residual and search direction stays in device memory (HBM);
  the operator is applied with its compiled plan (``smat_apply``) straight
  into preallocated buffers;
* the per-iteration scalar work (curvatures, step sizes, convergence and
  breakdown tests, soft thresholding, norms) runs as fused kernels of
  libsmat.so (csrc/solvers.cu) that keep their scalars in a small device state
  array, so an iteration needs no host round trip;
* CG solves all right-hand-side columns at once (the reference loops over
  columns, solvers.py:141-150); converged columns are frozen by their state;
* one iteration (applications + step kernels) is captured once in a CUDA
  graph and replayed; the host looks at the device state only every few
  iterations (doubling intervals) to stop early or raise.

Results come back as numpy arrays for numpy inputs (the reference contract)
and as device tensors for CUDA tensor inputs.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import (
    BreakdownError,
    DimensionMismatch,
    KOutOfRange,
    NegativeThreshold,
    NonSquare,
)

__all__ = [
    "IstaOptions", "IstaResult", "OmpResult", "SolveOptions", "SolveReport", "SpectralReport",
    "cg_solve", "ista", "omp", "power_iteration", "soft_threshold",
]


# ------------------------------------------------------------------ helpers --
def _torch():
    import torch

    if not torch.cuda.is_available():
        raise _native.NativeError("the solvers run on a CUDA device; none is available (no CPU fallback)")
    return torch


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _code(dtype) -> int:
    return _native.C128 if np.dtype(dtype) == np.complex128 else _native.F64


def _tdtype(dtype):
    torch = _torch()
    return torch.complex128 if np.dtype(dtype) == np.complex128 else torch.float64


def _np_of(x):
    """numpy dtype of a numpy array or torch tensor."""
    if _is_torch(x):
        import torch

        return np.dtype({torch.float32: np.float32, torch.float64: np.float64, torch.complex64: np.complex64,
                         torch.complex128: np.complex128, torch.int32: np.int32, torch.int64: np.int64,
                         torch.int16: np.int16, torch.int8: np.int8, torch.uint8: np.uint8,
                         torch.bool: np.bool_}.get(x.dtype, np.float64))
    return np.asarray(x).dtype


def _to_device(x, dtype, device):
    """(n,) or (n, K) input -> contiguous device tensor of the solver dtype."""
    torch = _torch()
    if _is_torch(x):
        return x.to(device=device, dtype=_tdtype(dtype)).contiguous()
    a = np.ascontiguousarray(np.asarray(x), dtype=dtype)
    return torch.from_numpy(a).to(device)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


# how the last solver loop ran: "graph" (captured once, replayed) or "eager"
last_loop_mode = None
# solver iterations replay one captured CUDA graph (tests flip this to compare
# against eager launches)
_GRAPHS = True


def _graphs_enabled() -> bool:
    return _GRAPHS


class _Loop:
    """Runs `body` (an iteration: plan applications + step kernels) either
    eagerly or as replays of one captured CUDA graph."""

    def __init__(self, body):
        self.body = body
        self.graph = None
        self.tried = False

    def run(self, count: int) -> None:
        torch = _torch()
        if count <= 0:
            return
        if not self.tried and _graphs_enabled() and count > 1:
            self.tried = True
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            # (a warm-up iteration outside the capture would change the state:
            # the plans' workspaces are allocated beforehand instead)
            try:
                with torch.cuda.stream(s):
                    with torch.cuda.graph(g, stream=s):
                        self.body()
                torch.cuda.current_stream().wait_stream(s)
                self.graph = g
            except Exception:  # capture unsupported here: run eagerly
                torch.cuda.current_stream().wait_stream(s)
                torch.cuda.synchronize()
                self.graph = None
        global last_loop_mode
        last_loop_mode = "graph" if self.graph is not None else "eager"
        for _ in range(count):
            if self.graph is not None:
                self.graph.replay()
            else:
                self.body()


class _Applier:
    """y = A x or A^H x through the compiled plan into preallocated buffers."""

    def __init__(self, op, dtype, ncols, device):
        self.op = op
        self.code, self.xcode = _native_work(op, dtype)
        self.plan = op._plan(self.code, device)
        self.ncols = ncols
        for d in (0, 1):
            # (this stream's workspaces; the capture stream's are allocated
            # inside the capture, from the graph's private pool)
            self.plan.workspace(d, ncols)

    def __call__(self, direction, x, y):
        from .core import _raw_stream

        torch = _torch()
        self.plan.apply_device(direction, x, self.xcode, y, self.ncols, _raw_stream(torch, x.device.index))


def _native_work(op, dtype):
    from .core import _work_codes

    pcode, xcode = _work_codes(op, np.dtype(dtype))
    if pcode != _code(dtype):
        raise _native.NativeError(f"solver dtype {np.dtype(dtype)} does not match the plan dtype code {pcode}")
    return pcode, xcode


def _scratch(n, k, device):
    torch = _torch()
    lib = _native.load_library()
    nbytes = int(lib.smat_solver_scratch_bytes(n, k))
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)


def _device_index():
    from .core import _default_device

    return _default_device()


def _out(t, like_torch):
    return t if like_torch else t.cpu().numpy()


# ---------------------------------------------------------- soft threshold --
def soft_threshold(x, c):
    """Shrink magnitudes toward zero by ``c`` (solvers.py:22-34): real entries
    map to sign(u)*max(|u|-c, 0), complex entries shrink in modulus keeping
    their phase.  Computed by a device kernel (float64 / complex128 result)."""
    if c < 0:
        raise NegativeThreshold(f"threshold must be >= 0, got {c}")
    like_torch = _is_torch(x) and x.is_cuda
    dt = np.complex128 if np.issubdtype(_np_of(x), np.complexfloating) else np.float64
    torch = _torch()
    dev = x.device if like_torch else torch.device("cuda", _device_index())
    src = _to_device(x, dt, dev)
    out = torch.empty_like(src)
    lib = _native.load_library()
    _native.check(lib.smat_soft_threshold(_code(dt), src.numel(), _ptr(src), _ptr(out), float(c), _stream()),
                  "smat_soft_threshold")
    return _out(out, like_torch)


# ------------------------------------------------------------------ CG -------
@dataclass
class SolveOptions:
    """Controls for :func:`cg_solve` (solvers.py:37-60)."""

    max_iterations: int | None = None
    relative_tolerance: float = 1e-10
    assume_hermitian: bool = False

    def __post_init__(self):
        if self.relative_tolerance <= 0:
            raise ValueError("relative_tolerance must be positive")
        if self.max_iterations is not None and self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")


@dataclass
class SolveReport:
    """Result of a linear solve (solvers.py:63-77); per-column fields collapse
    to scalars when the right-hand side was a single vector."""

    solution: np.ndarray
    iterations: np.ndarray
    residual_norm: np.ndarray
    converged: np.ndarray


def _check_intervals(max_iter):
    """Host checks of the device state after 4, 8, 16, ... 64 iterations."""
    done, step = 0, 4
    while done < max_iter:
        k = min(step, max_iter - done)
        yield k
        done += k
        step = min(step * 2, 64)


def cg_solve(A, y, options=None):
    """Solve A X = Y by conjugate gradients (solvers.py:109-160), all columns
    at once on the device.  One forward per iteration, plus one backward per
    iteration (and one on the right-hand side) in normal-equations mode."""
    options = options or SolveOptions()
    if A.rows != A.cols:
        raise NonSquare(f"cg_solve needs a square operator, got {A.shape}")
    if not _is_torch(y):
        y = np.asarray(y)
    like_torch = _is_torch(y) and y.is_cuda
    rhs_dt = _np_of(y)
    ndim = y.dim() if _is_torch(y) else np.asarray(y).ndim
    squeeze = ndim == 1
    rows_in = int(y.shape[0])
    if rows_in != A.rows:
        raise DimensionMismatch(f"right-hand side has {rows_in} rows, operator expects {A.rows}")
    max_iter = options.max_iterations or A.cols
    tol = options.relative_tolerance
    dtype = np.result_type(rhs_dt, A.field.dtype)
    torch = _torch()
    dev = y.device if like_torch else torch.device("cuda", _device_index())
    with torch.cuda.device(dev):
        rhs = _to_device(y, dtype, dev)
        if squeeze:
            rhs = rhs[:, None].contiguous()
        n, k = A.cols, rhs.shape[1]
        lib = _native.load_library()
        code = _code(dtype)
        ap_ = _Applier(A, dtype, k, dev.index)
        if options.assume_hermitian:
            b = rhs
        else:
            b = torch.empty_like(rhs)
            ap_(1, rhs, b)  # A^H y
        x = torch.empty_like(b)
        r = torch.empty_like(b)
        p = torch.empty_like(b)
        ap = torch.empty_like(b)
        tmp = torch.empty_like(b) if not options.assume_hermitian else None
        state = torch.zeros((k, _native.CG_STATE), dtype=torch.float64, device=dev)
        scratch = _scratch(n, k, dev)
        sb = scratch.numel()
        _native.check(lib.smat_cg_init(code, n, k, _ptr(b), _ptr(x), _ptr(r), _ptr(p), _ptr(state), float(tol),
                                       _ptr(scratch), sb, _stream()), "smat_cg_init")

        def body():
            if options.assume_hermitian:
                ap_(0, p, ap)
            else:
                ap_(0, p, tmp)
                ap_(1, tmp, ap)
            _native.check(lib.smat_cg_step(code, n, k, _ptr(x), _ptr(r), _ptr(p), _ptr(ap), _ptr(state),
                                           int(max_iter), _ptr(scratch), sb, _stream()), "smat_cg_step")

        loop = _Loop(body)
        st = state.cpu().numpy()
        for chunk in _check_intervals(max_iter):
            if np.all(st[:, 5] != 0):
                break
            loop.run(chunk)
            st = state.cpu().numpy()
            bad = np.nonzero(st[:, 5] == 2)[0]
            if bad.size:
                c = int(bad[0])
                raise BreakdownError(
                    f"non-positive curvature p^H A p = {st[c, 7]:.3e} at "
                    f"iteration {int(st[c, 4])}; operator is not positive definite"
                )
        iterations = st[:, 4].astype(int)
        residuals = st[:, 6].copy()
        converged = st[:, 5] == 1
    sol = x[:, 0] if squeeze else x
    sol = _out(sol, like_torch)
    if squeeze:
        return SolveReport(sol, int(iterations[0]), float(residuals[0]), bool(converged[0]))
    return SolveReport(sol, iterations, residuals, converged)


# ------------------------------------------------------------------ ISTA -----
@dataclass
class IstaOptions:
    """Controls for :func:`ista` (solvers.py:109-130)."""

    lam: float
    steps: int = 100
    step_size: float | None = None
    seed: int = 0

    def __post_init__(self):
        if self.lam <= 0:
            raise ValueError("lam must be positive")
        if self.steps < 1:
            raise ValueError("steps must be >= 1")
        if self.step_size is not None and self.step_size <= 0:
            raise ValueError("step_size must be positive")


@dataclass
class IstaResult:
    solution: np.ndarray
    objective_trace: np.ndarray
    step_size: float


def ista(M, b, options):
    """Iterative soft thresholding for min_x lam*||x||_1 + 0.5*||b - Mx||^2
    (solvers.py:163-194): ``steps`` iterations of
    ``x <- t_{lam*alpha}(x + alpha * M^H (b - M x))`` from ``x = 0``; the
    trace holds the objective of x_0 .. x_steps."""
    if not _is_torch(b):
        b = np.asarray(b)
    like_torch = _is_torch(b) and b.is_cuda
    ndim = b.dim() if _is_torch(b) else b.ndim
    if ndim != 1:
        raise ValueError("ista expects a single measurement vector")
    if int(b.shape[0]) != M.rows:
        raise DimensionMismatch(f"measurement has {int(b.shape[0])} rows, operator expects {M.rows}")
    alpha = options.step_size
    if alpha is None:
        spec = power_iteration(M, mode="singular", tol=1e-6, max_iter=50, seed=options.seed)
        alpha = 1.0 / (1.01 * spec.value ** 2)
    level = options.lam * alpha
    dtype = np.result_type(_np_of(b), M.field.dtype)
    torch = _torch()
    dev = b.device if like_torch else torch.device("cuda", _device_index())
    with torch.cuda.device(dev):
        lib = _native.load_library()
        code = _code(dtype)
        rhs = _to_device(b, dtype, dev)[:, None].contiguous()
        ap_ = _Applier(M, dtype, 1, dev.index)
        tdt = _tdtype(dtype)
        x = torch.zeros((M.cols, 1), dtype=tdt, device=dev)
        g = torch.empty_like(x)
        mx = torch.empty((M.rows, 1), dtype=tdt, device=dev)
        r = torch.empty_like(mx)
        trace = torch.zeros(options.steps + 1, dtype=torch.float64, device=dev)
        state = torch.zeros(2, dtype=torch.float64, device=dev)
        scratch = _scratch(max(M.rows, M.cols), 1, dev)
        sb = scratch.numel()
        lam = float(options.lam)

        def residual():
            ap_(0, x, mx)
            _native.check(lib.smat_ista_residual(code, M.rows, _ptr(rhs), _ptr(mx), _ptr(r), _ptr(trace),
                                                 _ptr(state), lam, _ptr(scratch), sb, _stream()),
                          "smat_ista_residual")

        def body():
            residual()
            ap_(1, r, g)
            _native.check(lib.smat_ista_update(code, M.cols, _ptr(x), _ptr(g), float(alpha), float(level),
                                               _ptr(state), _ptr(scratch), sb, _stream()), "smat_ista_update")

        _Loop(body).run(options.steps)
        residual()  # objective of the final iterate
        sol = x[:, 0]
        tr = trace.cpu().numpy()
    return IstaResult(_out(sol, like_torch), tr, float(alpha))


# ------------------------------------------------------------------- OMP -----
@dataclass
class OmpResult:
    """Greedy selection result (solvers.py:197-205)."""

    support: np.ndarray
    coefficients: np.ndarray
    solution: np.ndarray
    residual_norm: float


def omp(M, b, sparsity, residual_tol=None):
    """Orthogonal matching pursuit (solvers.py:208-261): correlate the
    residual through the device backward, pick the largest magnitude (lowest
    index on ties) with a device argmax, append the atom's column (one device
    forward of a unit vector) and re-fit the coefficients by a dense
    least-squares solve (QR) on the selected columns, all on the device."""
    if not _is_torch(b):
        b = np.asarray(b)
    like_torch = _is_torch(b) and b.is_cuda
    ndim = b.dim() if _is_torch(b) else b.ndim
    if ndim != 1:
        raise ValueError("omp expects a single measurement vector")
    if int(b.shape[0]) != M.rows:
        raise DimensionMismatch(f"measurement has {int(b.shape[0])} rows, operator expects {M.rows}")
    if not 1 <= sparsity <= M.cols:
        raise KOutOfRange(f"sparsity {sparsity} outside [1, {M.cols}]")
    dtype = np.result_type(_np_of(b), M.field.dtype)
    torch = _torch()
    dev = b.device if like_torch else torch.device("cuda", _device_index())
    with torch.cuda.device(dev):
        lib = _native.load_library()
        code = _code(dtype)
        tdt = _tdtype(dtype)
        rhs = _to_device(b, dtype, dev)[:, None].contiguous()
        ap_ = _Applier(M, dtype, 1, dev.index)
        stop_norm = residual_tol * float(torch.linalg.vector_norm(rhs)) if residual_tol is not None else None
        excluded = torch.zeros(M.cols, dtype=torch.uint8, device=dev)
        corr = torch.empty((M.cols, 1), dtype=tdt, device=dev)
        unit = torch.zeros((M.cols, 1), dtype=tdt, device=dev)
        atom_idx = torch.zeros(1, dtype=torch.int64, device=dev)
        scratch = _scratch(max(M.rows, M.cols), 1, dev)
        columns = torch.empty((M.rows, 0), dtype=tdt, device=dev)
        coeffs = torch.zeros(0, dtype=tdt, device=dev)
        residual = rhs.clone()
        support = []
        for _ in range(sparsity):
            ap_(1, residual, corr)
            _native.check(lib.smat_abs_argmax(code, M.cols, _ptr(corr), _ptr(excluded), _ptr(atom_idx),
                                              _ptr(scratch), scratch.numel(), _stream()), "smat_abs_argmax")
            atom = int(atom_idx.item())
            support.append(atom)
            excluded[atom] = 1
            unit.zero_()
            unit[atom, 0] = 1
            col = torch.empty((M.rows, 1), dtype=tdt, device=dev)
            ap_(0, unit, col)
            columns = torch.cat([columns, col], dim=1)
            q, rr = torch.linalg.qr(columns)
            coeffs = torch.linalg.solve_triangular(rr, q.conj().T @ rhs, upper=True)[:, 0]
            residual = rhs - columns @ coeffs[:, None]
            if stop_norm is not None and float(torch.linalg.vector_norm(residual)) <= stop_norm:
                break
        solution = torch.zeros(M.cols, dtype=tdt, device=dev)
        solution[torch.as_tensor(support, device=dev)] = coeffs
        res_norm = float(torch.linalg.vector_norm(residual))
    return OmpResult(np.asarray(support, dtype=int), _out(coeffs, like_torch), _out(solution, like_torch),
                     res_norm)


# ------------------------------------------------------- power iteration -----
@dataclass
class SpectralReport:
    """Dominant eigen/singular estimate (solvers.py:264-274)."""

    value: float
    vector: np.ndarray
    iterations: int
    converged: bool


def power_iteration(A, mode="eigen", tol=1e-9, max_iter=1000, seed=0):
    """Largest-magnitude eigenvalue (``mode='eigen'``) or largest singular
    value (``mode='singular'``, iterates on A^H A) by the power method from the
    reference's seeded random start (solvers.py:277-333).  Non-convergence is
    reported through ``converged``."""
    if mode not in ("eigen", "singular"):
        raise ValueError(f"mode must be 'eigen' or 'singular', got {mode!r}")
    if mode == "eigen" and A.rows != A.cols:
        raise NonSquare(f"eigen mode needs a square operator, got {A.shape}")
    rng = np.random.default_rng(seed)
    n = A.cols
    v0 = rng.standard_normal(n)
    if A.field.dtype == np.complex128:
        v0 = v0 + 1j * rng.standard_normal(n)
    v0 = v0 / np.linalg.norm(v0)
    dtype = v0.dtype
    torch = _torch()
    dev = torch.device("cuda", _device_index())
    with torch.cuda.device(dev):
        lib = _native.load_library()
        code = _code(dtype)
        ap_ = _Applier(A, dtype, 1, dev.index)
        v = torch.from_numpy(np.ascontiguousarray(v0)).to(dev)[:, None].contiguous()
        w = torch.empty_like(v)
        tmp = torch.empty((A.rows, 1), dtype=v.dtype, device=dev) if mode == "singular" else None
        state = torch.zeros(6, dtype=torch.float64, device=dev)
        scratch = _scratch(max(A.rows, A.cols), 1, dev)
        sb = scratch.numel()

        def body():
            if mode == "eigen":
                ap_(0, v, w)
            else:
                ap_(0, v, tmp)
                ap_(1, tmp, w)
            _native.check(lib.smat_power_step(code, n, _ptr(v), _ptr(w), _ptr(state), float(tol), _ptr(scratch), sb,
                                              _stream()), "smat_power_step")

        loop = _Loop(body)
        st = state.cpu().numpy()
        for chunk in _check_intervals(max_iter):
            loop.run(chunk)
            st = state.cpu().numpy()
            if st[2] != 0:
                break
        vec = v[:, 0].cpu().numpy()
    its = int(st[1])
    if st[5] != 0:  # operator annihilated the iterate
        return SpectralReport(0.0, vec, its, True)
    est = float(st[0])
    value = np.sqrt(est) if mode == "singular" else est
    if st[3] != 0:
        return SpectralReport(float(value), vec, its, True)
    return SpectralReport(float(value), vec, max_iter, False)
