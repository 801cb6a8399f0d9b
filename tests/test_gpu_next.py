"""Parity of the SURVEY §8(f) rows built on the same kernels (C-ABI vs oracle).

NEXT-1 (QMR dual GEMV): A·p and Aᴴ·q of one QMR iteration from ONE pass over A
(gemv_cols<DO_N, DO_H>).  The column-owner layout is also selectable for A·x
alone (CCG_GEMV=cols), checked here against the oracle's product with the
same per-matvec bar as test_gpu_apply.py.
"""

import numpy as np
import pytest

import oracle
from oracle import DenseOp
from oracle.operators import reference_apply
from workloads import dense_random, cfg2, gauss_shifted_rows, cfg3_rhs
from tests._gpu import Dense, TOL, XTOL, relerr

pytestmark = pytest.mark.gpu


def _x(n, dtype, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(dtype)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("n", [2, 8, 31, 64, 257, 1000, 2048, 4097])
def test_cols_gemv_apply(monkeypatch, dtype, n):
    """A·x through the column-owner kernel + strip sum (ragged tails: n not a
    multiple of the 256·V-column strip or of the 8-row group)."""
    if dtype == np.complex64 and n % 2:
        n += 1                                   # cols layout needs n % V == 0 (else old path)
    monkeypatch.setenv("CCG_GEMV", "cols")
    A = dense_random(n, seed=n, dtype=dtype, shift=1.0 + 0.5j)
    x = _x(n, dtype, seed=n + 1)
    with Dense(A) as h:
        y = h.apply(x, "A")
        y2 = h.apply(x, "A")
    assert relerr(y, reference_apply(A, x, "A")) <= TOL[dtype]
    assert np.array_equal(y, y2)                 # deterministic


@pytest.mark.parametrize("dual", ["0", "1"])
@pytest.mark.parametrize("n", [1, 7, 257, 1000, 2050])
def test_qmr_dual_ragged(monkeypatch, dual, n):
    monkeypatch.setenv("CCG_QMR_DUAL", dual)
    A = dense_random(n, seed=n, dtype=np.complex128, shift=3 - 1j)
    y = dense_random(n, seed=n + 1)[:, 0] * 3
    o = oracle.solve("qmr", DenseOp(A), y, 1e-10, 400)
    with Dense(A) as h:
        g = h.solve("qmr", y, 1e-10, 400)
        assert g["status"] == "CONVERGED" and abs(g["iterations"] - o.iterations) <= 2
        assert (g["matvecs_a"], g["matvecs_ah"]) == (o.matvecs_a, o.matvecs_ah)
        k = min(g["iterations"], o.iterations)
        ge = h.solve("qmr", y, 0.0, k)
    oe = oracle.solve("qmr", DenseOp(A), y, 0.0, k)
    assert relerr(ge["x"], oe.x) <= XTOL[np.complex128]


def test_qmr_dual_cfg2(monkeypatch):
    """BASELINE config 2 (n = 4096 c128, DDA lattice): QMR through the dual GEMV,
    P-literal (±2 iterations, x at equal k within 1e-9)."""
    monkeypatch.setenv("CCG_QMR_DUAL", "1")
    A, y = cfg2()
    o = oracle.solve("qmr", DenseOp(A), y, 1e-8, 1000)
    with Dense(A) as h:
        g = h.solve("qmr", y, 1e-8, 1000)
        assert g["status"] == "CONVERGED" and abs(g["iterations"] - o.iterations) <= 2
        assert g["true_rel_res"] <= 1e-7
        k = min(g["iterations"], o.iterations)
        ge = h.solve("qmr", y, 0.0, k)
    oe = oracle.solve("qmr", DenseOp(A), y, 0.0, k)
    assert relerr(ge["x"], oe.x) <= 1e-9


def test_qmr_dual_c64_proxy(monkeypatch):
    monkeypatch.setenv("CCG_QMR_DUAL", "1")
    n = 4096
    A = gauss_shifted_rows(n, 0, n, seed=1)
    y = cfg3_rhs(n)
    o = oracle.solve("qmr", DenseOp(A), y, 1e-5, 500)
    with Dense(A) as h:
        g = h.solve("qmr", y, 1e-5, 500)
        assert g["status"] == "CONVERGED" and abs(g["iterations"] - o.iterations) <= 2
        k = min(g["iterations"], o.iterations)
        ge = h.solve("qmr", y, 0.0, k)
    oe = oracle.solve("qmr", DenseOp(A), y, 0.0, k)
    assert relerr(ge["x"], oe.x) <= XTOL[np.complex64]
