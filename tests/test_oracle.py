"""Pin the CPU oracle (oracle/linop_oracle.py) before trusting it.

Checked against (a) the reference's own known-answer tests
(reference tests/test_kernels.py, tests/test_leaves.py) and (b) the golden
fixtures recorded from the real reference package (tests/golden/make_golden.py).
Bit-exact where the reference is (FWHT, and the FFT paths, which follow the
same operation order), tolerance elsewhere.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import ref_close, rel_l2
from oracle import linop_oracle as orc


def _keys(d, prefix):
    return sorted({k.split("/")[1] for k in d if k.startswith(prefix + "/")})


# ------------------------------------------------ known-answer tests -------
def test_fwht_known_vector():
    # reference tests/test_kernels.py:74-75
    assert np.array_equal(orc.fwht([1, 2, 3, 4]), [10, -2, -4, 0])


def test_fwht_impulse_and_length_one():
    x = np.zeros(8)
    x[0] = 1
    assert np.array_equal(orc.fwht(x), np.ones(8))  # tests/test_kernels.py:69-72
    assert np.array_equal(orc.fwht([7.0]), [7.0])  # :66-67


def test_fwht_matches_sylvester_and_involution():
    for order in range(7):
        h = np.array([[1.0]])
        for _ in range(order):
            h = np.block([[h, h], [h, -h]])
        x = np.random.default_rng(order).standard_normal(1 << order)
        assert ref_close(orc.fwht(x), h @ x)[0]
        assert ref_close(orc.fwht(orc.fwht(x)), (1 << order) * x)[0]


def test_dft_known_answers():
    # reference tests/test_kernels.py:16-23
    assert ref_close(orc.dft([1, 0, 0, 0]), np.ones(4))[0]
    assert ref_close(orc.dft([1, 1, 1, 1]), [4, 0, 0, 0])[0]
    assert ref_close(orc.dft([0, 1, 0, 0]), [1, -1j, -1, 1j])[0]


@pytest.mark.parametrize("n", list(range(1, 18)) + [32, 100, 128])
def test_dft_matches_definition(n):
    x = np.random.default_rng(n).standard_normal(n) + 1j
    j = np.arange(n)
    F = np.exp(-2j * np.pi * np.outer(j, j) / n)
    assert ref_close(orc.dft(x), F @ x)[0]
    assert np.max(np.abs(orc.dft(orc.dft(x), inverse=True) - x)) <= 1e-12 * np.linalg.norm(x)


def test_circulant_and_toeplitz_small_known():
    # Circulant([0,1,0]).forward([5,6,7]) = [7,5,6] (tests/test_leaves.py:176-177)
    assert ref_close(orc.apply(orc.circulant([0.0, 1.0, 0.0]), [5.0, 6.0, 7.0]), [7, 5, 6])[0]
    # Toeplitz([1,2],[3]) -> [[1,3],[2,1]], forward [4,3] (tests/test_leaves.py:210-213)
    t = orc.toeplitz([1.0, 2.0], [3.0])
    assert ref_close(orc.to_dense(t), [[1, 3], [2, 1]])[0]
    assert ref_close(orc.apply(t, [1.0, 1.0]), [4, 3])[0]


# ------------------------------------------------------ golden fixtures -----
def test_golden_kernels(golden_kernels):
    g = golden_kernels
    for n in _keys(g, "dft"):
        x = g[f"dft/{n}/x"]
        assert np.array_equal(orc.dft(x), g[f"dft/{n}/fwd"]), n
        assert np.array_equal(orc.dft(x, inverse=True), g[f"dft/{n}/inv"]), n
    for o in _keys(g, "fwht"):
        assert np.array_equal(orc.fwht(g[f"fwht/{o}/x"]), g[f"fwht/{o}/y"]), o
    for n in _keys(g, "cconv"):
        c, x = g[f"cconv/{n}/c"], g[f"cconv/{n}/x"]
        got = orc.apply(orc.circulant(c), x)
        assert rel_l2(got, g[f"cconv/{n}/y"]) <= 1e-14, n


def _check_fb(g, key, op, exact=True, tol=1e-13):
    fx = orc.apply(op, g[f"{key}/x"], 0)
    by = orc.apply(op, g[f"{key}/y"], 1)
    if exact:
        assert np.array_equal(fx, g[f"{key}/fwd"]), key
        assert np.array_equal(by, g[f"{key}/bwd"]), key
    else:
        assert rel_l2(fx, g[f"{key}/fwd"]) <= tol, key
        assert rel_l2(by, g[f"{key}/bwd"]) <= tol, key


def test_golden_hadamard_bit_exact(golden_ops):
    g = golden_ops
    for o in _keys(g, "hadamard"):
        order = int(o.split("=")[1])
        _check_fb(g, f"hadamard/{o}", orc.hadamard(order))
        xi = g[f"hadamard_i32/{o}/x"]
        assert np.array_equal(orc.apply(orc.hadamard(order), xi), g[f"hadamard_i32/{o}/y"])
    h = orc.hadamard(10)
    assert np.array_equal(orc.apply(h, g["c1/X"]), g["c1/fwd"])
    assert np.array_equal(orc.apply(h, g["c1/X"], 1), g["c1/bwd"])
    assert np.array_equal(orc.apply(h, g["c1/Xi"]), g["c1/fwd_i32"])
    # int32 C1 result is exactly integral and equals the int64 dense product
    assert np.array_equal(g["c1/fwd_i32"], np.round(g["c1/fwd_i32"]))


def test_golden_fourier_circulant(golden_ops):
    g = golden_ops
    for n in _keys(g, "fourier"):
        _check_fb(g, f"fourier/{n}", orc.fourier(int(n.split("=")[1])))
    for kind in ("circulant_rr", "circulant_cc"):
        for n in _keys(g, kind):
            key = f"{kind}/{n}"
            _check_fb(g, key, orc.circulant(g[f"{key}/c"]))


def test_golden_toeplitz(golden_ops):
    g = golden_ops
    for i in _keys(g, "toeplitz"):
        key = f"toeplitz/{i}"
        _check_fb(g, key, orc.toeplitz(g[f"{key}/col"], g[f"{key}/row"]))


def test_golden_kron(golden_ops):
    g = golden_ops
    for i, (o, f, c) in enumerate([(1, 2, 4), (2, 4, 8), (3, 8, 16)]):
        key = f"kron/{i}"
        op = orc.kron(orc.hadamard(o), orc.fourier(f), orc.circulant(g[f"{key}/c"]))
        _check_fb(g, key, op, exact=False, tol=1e-14)


def test_golden_c5_chain(golden_ops):
    g = golden_ops
    for n in _keys(g, "c5"):
        key = f"c5/{n}"
        N = int(n.split("=")[1])
        op = orc.chain_c5(N, g[f"{key}/d1"], g[f"{key}/d2"], g[f"{key}/U"], g[f"{key}/V"])
        _check_fb(g, key, op, exact=False, tol=1e-13)


def test_config_check_record_present():
    """The full-size reference-vs-oracle check (make_golden.py --config-check)
    was run and found the oracle bit-exact (C1-C4) / within 1e-15 (C5)."""
    from conftest import GOLDEN

    text = (GOLDEN / "config_check.txt").read_text()
    for name in ("C1 f64", "C1 int32", "C2", "C3", "C4", "C5"):
        assert name in text
    for line in text.splitlines():
        fwd = float(line.split("relL2 fwd ")[1].split()[0])
        bwd = float(line.split(" bwd ")[1].split()[0])
        assert fwd <= 1e-14 and bwd <= 1e-14, line
