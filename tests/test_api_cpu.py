"""Host-side behaviour that needs no GPU: the library loads and exports every
symbol of include/smat.h, validation mirrors the reference (errors.py, core.py),
dtype/field promotion, serialisation of the operator tree, footprints, and
that the product path refuses to run (loudly) without a CUDA device."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1710_09578_b200 as sm
from paper_1710_09578_b200 import _native
from paper_1710_09578_b200.core import _work_codes

REPO = Path(__file__).resolve().parent.parent


def test_library_exports_every_header_symbol():
    header = (REPO / "include" / "smat.h").read_text()
    declared = set(re.findall(r"SMAT_API\s+[\w\s\*]+?\b(smat_\w+)\s*\(", header))
    assert declared == set(_native.EXPORTED_SYMBOLS)
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    assert _native.load_library().smat_abi_version() == 3


def test_block_layout_classification():
    """Strided views reach the engine with their leading dimension (no copy):
    column slices of a wider row-major block, and column-major blocks."""
    from paper_1710_09578_b200.core import _block_layout

    assert _block_layout(8, 1, 100, 8) == (0, _native.ROW_MAJOR)          # dense
    assert _block_layout(64, 1, 100, 8) == (64, _native.ROW_MAJOR)        # column slice
    assert _block_layout(64, 0, 100, 1) == (64, _native.ROW_MAJOR)        # one column of a block
    assert _block_layout(1, 100, 100, 8) == (100, _native.COL_MAJOR)      # Fortran order
    assert _block_layout(1, 128, 100, 8) == (128, _native.COL_MAJOR)      # slice of a Fortran block
    assert _block_layout(2, 3, 100, 8)[0] == -1                           # neither: dense copy
    assert _block_layout(-8, 1, 100, 8)[0] == -1                          # negative stride


def test_struct_layout_matches_header():
    # smat_param: ptr + i64 + 2*i32 = 24 bytes; smat_node = 4*i32 + 2*i64 + 4*i64 + 2*f64 + 4*param
    assert ctypes.sizeof(_native.SmatParam) == 24
    assert ctypes.sizeof(_native.SmatNode) == 16 + 16 + 32 + 16 + 4 * 24


def test_no_cuda_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(_native.NativeError, match="no CPU fallback"):
        sm.Hadamard(3).forward(np.ones(8))


# ------------------------------------------------------------ validation ----
def test_dimension_mismatch_messages():
    with pytest.raises(sm.DimensionMismatch) as info:
        sm.Identity(4).forward(np.zeros(3))
    msg = str(info.value)
    assert "(4, 4)" in msg and "3" in msg
    with pytest.raises(sm.DimensionMismatch):
        sm.Zero(2, 3).backward(np.zeros(3))
    assert issubclass(sm.DimensionMismatch, ValueError)


def test_type_and_ndim_errors():
    with pytest.raises(TypeError):
        sm.Identity(2).forward(np.array(["a", "b"], dtype=object))
    with pytest.raises(ValueError):
        sm.Identity(2).forward(np.zeros((2, 2, 2)))


def test_constructor_errors_match_reference():
    with pytest.raises(sm.OrderTooLarge):
        sm.Hadamard(31)
    with pytest.raises(ValueError):
        sm.Hadamard(-1)
    with pytest.raises(sm.EmptyInput):
        sm.Diagonal([])
    with pytest.raises(sm.EmptyInput):
        sm.Circulant([])
    with pytest.raises(sm.EmptyInput):
        sm.Toeplitz([])
    with pytest.raises(sm.EmptyInput):
        sm.Dense(np.zeros((0, 3)))
    with pytest.raises(ValueError):
        sm.Zero(0, 3)
    with pytest.raises(sm.ChainMismatch) as info:
        sm.Product(sm.Zero(2, 3), sm.Zero(4, 2))
    assert "(2, 3)" in str(info.value) and "(4, 2)" in str(info.value)
    with pytest.raises(sm.EmptyInput):
        sm.Product()
    with pytest.raises(sm.TooFewFactors):
        sm.Kron(sm.Identity(2))
    with pytest.raises(sm.IndexOutOfRange):
        sm.Partial(sm.Identity(3), row_indices=[3])
    with pytest.raises(sm.IndexOutOfRange):
        sm.Partial(sm.Identity(3), col_indices=[-1])
    with pytest.raises(sm.RaggedGrid):
        sm.Blocks([[sm.Identity(2), sm.Identity(2)], [sm.Identity(2)]])
    with pytest.raises(sm.BlockShapeMismatch) as info:
        sm.Blocks([[sm.Identity(2), sm.Identity(3)]])
    assert "(0,1)" in str(info.value)
    with pytest.raises(sm.BlockShapeMismatch):
        sm.Sum(sm.Identity(2), sm.Identity(3))
    with pytest.raises(sm.NotPowerOfTwo):
        sm.fwht(np.zeros(6))
    with pytest.raises(sm.EmptyInput):
        sm.dft(np.zeros(0))
    with pytest.raises(sm.DimensionMismatch):
        sm.DftPlan(8).execute(np.zeros(9))
    with pytest.raises(sm.DimensionMismatch):
        sm.circular_convolve([1, 0], [1, 0, 0])


def test_kron_overflow_guard():
    big = sm.Zero(1 << 21, 1 << 21)
    with pytest.raises(OverflowError):
        sm.Kron(big, big, big, big)


# --------------------------------------------------------------- fields -----
def test_field_lattice_and_aliases():
    R, C = sm.ScalarField.REAL64, sm.ScalarField.COMPLEX128
    assert sm.promote_field(R, C) is C and sm.promote_field(R, R) is R
    assert sm.as_field(np.float32) is R and sm.as_field(np.complex64) is C
    assert sm.as_field("complex128") is C
    with pytest.raises(ValueError):
        sm.as_field("float16ish")
    assert sm.Diag is sm.Diagonal and sm.Matrix is sm.Dense
    h = sm.Hadamard(4)
    assert (h.numN, h.numM) == h.shape == (16, 16)
    assert sm.Fourier(4).field is C and sm.Hadamard(2).field is R
    assert isinstance(h.H, sm.Adjoint) and h.H.H is h
    assert sm.Toeplitz([1.0, 2.0], [3.0, 4.0]).shape == (2, 3)


def test_working_precision_codes():
    F32, F64, C64, C128, I32, I64 = range(6)
    assert _work_codes(sm.Hadamard(3), np.dtype(np.int32)) == (I32, I32)
    assert _work_codes(sm.Hadamard(3), np.dtype(np.int64)) == (I64, I64)
    assert _work_codes(sm.Hadamard(3), np.dtype(np.int16)) == (F64, F64)
    assert _work_codes(sm.Fourier(4), np.dtype(np.int32)) == (C128, F64)
    assert _work_codes(sm.Fourier(4), np.dtype(np.float32)) == (C64, F32)
    assert _work_codes(sm.Circulant([1.0, 2.0]), np.dtype(np.float32)) == (F32, F32)
    assert _work_codes(sm.Circulant([1.0, 2.0]), np.dtype(np.complex64)) == (C64, C64)
    assert _work_codes(sm.Circulant([1j, 2.0]), np.dtype(np.float64)) == (C128, F64)
    assert _work_codes(sm.Kron(sm.Hadamard(1), sm.Identity(2)), np.dtype(np.int32)) == (I32, I32)
    assert _work_codes(sm.Kron(sm.Hadamard(1), sm.Diag([1, 2])), np.dtype(np.int32)) == (F64, F64)


def test_footprints():
    assert sm.Fourier(4096).footprint_bytes() <= 64
    assert sm.Zero(2, 3).footprint_bytes() <= 64
    k = 100
    fp = sm.Diagonal(np.ones(k, dtype=np.complex128)).footprint_bytes()
    assert 16 * k <= fp <= 16 * k + 64
    ks = np.array([8, 16, 32, 64])
    fps = [sm.Kron(sm.Fourier(int(k)), sm.Diag(np.ones(k) + 1j), sm.Dense(np.ones((k, k)) + 1j)).footprint_bytes()
           for k in ks]
    slope = np.polyfit(np.log(ks), np.log(fps), 1)[0]
    assert 1.8 <= slope <= 2.2
    s = sm.Dense(np.ones((4, 4)))
    z = sm.Zero(4, 4)
    shared = sm.Blocks([[s, z], [z, s]])
    separate = sm.Blocks([[sm.Dense(np.ones((4, 4))), z], [z, sm.Dense(np.ones((4, 4)))]])
    assert shared.footprint_bytes() < separate.footprint_bytes()


def test_to_dense_cap():
    with pytest.raises(sm.MaterializationTooLarge):
        sm.Zero(1 << 16, 1 << 16).to_dense()
    with pytest.raises(sm.MaterializationTooLarge):
        sm.Zero(64, 64).to_dense(cap_bytes=64 * 64 * 8)


# -------------------------------------------------------- serialisation -----
def test_serializer_shares_repeated_subtrees():
    s = sm.Dense(np.ones((3, 3)))
    op = sm.Blocks([[s, s], [s, sm.Identity(3)]])
    ser = _native.Serializer()
    root = ser.emit(op)
    kinds = [r["kind"] for r in ser.records]
    assert kinds.count(_native.DENSE) == 1 and kinds.count(_native.IDENTITY) == 1
    assert ser.records[root]["kind"] == _native.BLOCKS
    assert ser.records[root]["n_children"] == 4
    nodes, kids = ser.arrays()
    assert nodes[root].iparam[0] == 2 and nodes[root].iparam[1] == 2
    assert list(kids)[:4] == [0, 0, 0, 1]


def test_serializer_params_and_shapes():
    c5 = sm.Product(sm.Diag(np.ones(5) + 0j), sm.Fourier(5), sm.Diag(np.ones(5)),
                    sm.Sum(sm.Partial(sm.Hadamard(3), np.arange(5), np.arange(5)),
                           sm.LowRank(np.ones((5, 2)), np.ones((5, 2)))))
    ser = _native.Serializer()
    root = ser.emit(c5)
    nodes, _ = ser.arrays()
    assert nodes[root].kind == _native.PRODUCT and nodes[root].n_children == 4
    lr = [n for n in nodes if n.kind == _native.LOWRANK][0]
    assert lr.iparam[0] == 2 and lr.param[0].len == 10 and lr.param[2].len == 0
    part = [n for n in nodes if n.kind == _native.PARTIAL][0]
    assert list(part.iparam) == [1, 1, 1, 1] and part.param[0].dtype == _native.I64


def test_operator_algebra_sugar():
    a, b = sm.Fourier(4), sm.Hadamard(2)
    assert isinstance(a @ b, sm.Product) and isinstance(a * b, sm.Product)
    assert isinstance(a + b, sm.Sum) and (a + b).field is sm.ScalarField.COMPLEX128


def test_bench_reference_arm_json_cpu():
    """`bench.py --impl reference` runs the unmodified reference package
    (baseline/_ref, else /root/reference) on the host (no GPU needed) and
    prints the contract's JSON line."""
    import json
    import subprocess
    import sys

    root = Path(__file__).resolve().parent.parent
    res = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--workload", "c1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "reference" and "linopkit" in line["cpu_baseline"]["sample"]


