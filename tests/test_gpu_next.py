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


# ---------------------------------------------------------------------------
# NEXT-3: BiCG, CGS, CGNR (§2.1), COCR (§3.4) through ccg_solve
# ---------------------------------------------------------------------------
import paper_1208_4869_b200 as ccg                       # noqa: E402
from oracle import CsrOp                                   # noqa: E402
from oracle.solvers import NEXT3 as _N3, NEXT2              # noqa: E402
NEXT3 = _N3 + NEXT2          # the generic per-method GPU checks cover NEXT-2 (iii) too
from workloads import cfg1, helmholtz_csr, helmholtz_rhs   # noqa: E402
from tests._gpu import Csr                                 # noqa: E402
from tests.test_gpu_solve import _parity, _record          # noqa: E402


def _csym(A):
    return ((A + A.T) / 2).astype(A.dtype)


@pytest.mark.parametrize("method", NEXT3)
def test_next3_cfg1(method):
    A, y = cfg1()
    if method == "cocr":
        A = _csym(A)              # COCR is defined for complex-symmetric A
    with Dense(A) as h:
        o, g = _parity(h, DenseOp(A), y, method, 1e-10, 500, np.complex128, tag="cfg1-next3")
        assert (g["matvecs_a"], g["matvecs_ah"]) == (o.matvecs_a, o.matvecs_ah)
        h.solve(method, y, 1e-10, 500)
        hist = ccg.ccg_get_history(h.h)
        np.testing.assert_allclose(hist, np.array(o.history, float) / o.history[0], rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("method", NEXT3)
def test_next3_cfg2(method):
    """BASELINE config 2 (complex-symmetric DDA lattice, the natural COCR case)."""
    A, y = cfg2()
    with Dense(A) as h:
        _parity(h, DenseOp(A), y, method, 1e-8, 2000, np.complex128, tag="cfg2-next3",
                literal=method in ("bicg", "cocr"))


@pytest.mark.parametrize("method", ["bicg", "cgs", "cgnr", "tfqmr", "pbicgstab"])
def test_next3_cfg3_proxy_c64(method):
    n = 4096
    A = gauss_shifted_rows(n, 0, n, seed=1)
    y = cfg3_rhs(n)
    with Dense(A) as h:
        _parity(h, DenseOp(A), y, method, 1e-5, 500, np.complex64, tag="cfg3-proxy-next3", literal=False)


@pytest.mark.parametrize("n", [1, 7, 257, 1000])
@pytest.mark.parametrize("method", NEXT3)
def test_next3_ragged(method, n):
    A = dense_random(n, seed=n, dtype=np.complex128, shift=3 - 1j)
    if method == "cocr":
        A = _csym(A)
    y = dense_random(n, seed=n + 1)[:, 0] * 3
    with Dense(A) as h:
        _parity(h, DenseOp(A), y, method, 1e-10, 600, np.complex128, tag=f"ragged{n}-next3")


@pytest.mark.parametrize("method", NEXT3)
def test_next3_degenerate(method):
    c = 3 - 4j
    n = 10
    y = (np.arange(n) + 1j * np.arange(n)[::-1]).astype(np.complex128)
    with Dense(c * np.eye(n, dtype=np.complex128)) as h:
        g = h.solve(method, y, 1e-12, 50)
    assert g["status"] == "CONVERGED" and g["iterations"] == 1
    np.testing.assert_allclose(g["x"], y / c, rtol=1e-14, atol=1e-14)
    A, yy = cfg1(n=32, seed=2)
    if method == "cocr":
        A = _csym(A)
    with Dense(A) as h:
        g = h.solve(method, np.zeros(32, np.complex128), 1e-10, 10)
        assert g["status"] == "CONVERGED" and g["iterations"] == 0
        g = h.solve(method, yy, 0.0, 3)
        o = oracle.solve(method, DenseOp(A), yy, 0.0, 3)
        assert g["status"] == "MAXIT" and g["iterations"] == 3
        assert (g["matvecs_a"], g["matvecs_ah"]) == (o.matvecs_a, o.matvecs_ah)
        yb = yy.copy()
        yb[5] = np.nan
        assert h.solve(method, yb, 1e-10, 10)["status"] == "NONFINITE"
        xs = np.linalg.solve(A, yy)
        o = oracle.solve(method, DenseOp(A), yy, 1e-12, 200, x0=0.5 * xs)
        g = h.solve(method, yy, 1e-12, 200, x0=0.5 * xs)
        assert abs(g["iterations"] - o.iterations) <= 2 and relerr(g["x"], o.x) <= 1e-9


def test_next3_breakdown_fixture():
    A = np.array([[0, 1], [-1, 0]], dtype=np.complex128)
    y = np.array([1, 0], dtype=np.complex128)
    with Dense(A) as h:
        for m, name in (("bicg", "sigma"), ("cgs", "sigma"), ("cocr", "rho"), ("tfqmr", "sigma"),
                        ("bicgstabl", "sigma"), ("pbicgstab", "sigma")):
            g = h.solve(m, y, 1e-10, 10)
            o = oracle.solve(m, DenseOp(A), y, 1e-10, 10)
            assert g["status"] == "BREAKDOWN" and g["breakdown"] == name == o.breakdown, m
            assert g["iterations"] == o.iterations == 0, m
        g = h.solve("cgnr", y, 1e-10, 10)
        assert g["status"] == "CONVERGED" and g["iterations"] == 1


@pytest.mark.parametrize("method", ["cgs", "cocr", "tfqmr", "gmres", "pbicgstab"])
def test_next3_csr_transpose_free(method):
    """CGS and COCR need only A·x: they run on a CSR operator without the
    symmetric flag (COCR on the complex-symmetric shifted Helmholtz matrix)."""
    N = 16
    rp, ci, v = helmholtz_csr(N, kh=10 / 128)
    y = helmholtz_rhs(N)
    with Csr(rp, ci, v, N ** 3) as h:
        _parity(h, CsrOp(rp, ci, v), y, method, 1e-8, 3000, np.complex128, literal=False, tag="csr-next3")


def test_next3_csr_capability():
    rp, ci, v = helmholtz_csr(6)
    with Csr(rp, ci, v, 216) as h:
        for m in ("bicg", "cgnr"):
            with pytest.raises(ccg.CcgError) as e:
                h.solve(m, np.ones(216, np.complex128), 1e-8, 10)
            assert e.value.code == -3
    with Csr(rp, ci, v, 216, flags=ccg.FLAG_SYMMETRIC) as h:
        g = h.solve("bicg", helmholtz_rhs(6), 1e-8, 500)
        assert g["status"] == "CONVERGED"


# ---------------------------------------------------------------------------
# NEXT-4: matrix-free 7-point stencil operator (ccg_set_matvec_stencil7)
# ---------------------------------------------------------------------------
from workloads import lattice_csr, helmholtz_coeffs          # noqa: E402
from tests._gpu import to_dev, dt_name                         # noqa: E402
import torch                                                   # noqa: E402


class Stencil(Dense):
    def __init__(self, nx, ny, nz, d, ox, oy=None, oz=None, dtype=np.complex128):
        self.n = nx * ny * nz
        self.dtype = dtype
        self.h = ccg.ccg_create(dt_name(dtype), self.n)
        ccg.ccg_set_matvec_stencil7(self.h, nx, ny, nz, d, ox, oy, oz)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 3, 4), (33, 9, 5), (64, 7, 3), (31, 17, 12), (128, 8, 9)])
def test_stencil_apply_parity(dtype, dims):
    nx, ny, nz = dims
    d, ox, oy, oz = 5.5 - 0.25j, -1.0 + 0.125j, -0.5, 0.75j
    op = CsrOp(*lattice_csr(nx, ny, nz, d, ox, oy, oz, dtype=dtype))
    x = _x(nx * ny * nz, dtype, seed=nx)
    with Stencil(nx, ny, nz, d, ox, oy, oz, dtype=dtype) as h:
        for o in ("A", "AH", "AT"):
            assert relerr(h.apply(x, o), reference_apply(op, x, o)) <= TOL[dtype], o


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("dims", [(1, 1, 1), (1, 5, 1), (2, 3, 4), (33, 9, 5), (31, 17, 12), (128, 8, 9), (65, 10, 17)])
def test_stencil_apply_parity_real_offdiagonals(dtype, dims):
    """Real ox, oy, oz (a Laplacian-type operator, as config 5's) run the REALO
    kernel variant (matvec.cuh stencil7_kernel: the FMAs by the zero imaginary
    part are skipped): same parity bar at ragged sizes, and — the CSR kernel
    keeps those FMAs — equal values element by element."""
    nx, ny, nz = dims
    d, ox, oy, oz = 5.5 - 0.25j, -1.0, -0.5, 0.75
    rp, ci, v = lattice_csr(nx, ny, nz, d, ox, oy, oz, dtype=dtype)
    op = CsrOp(rp, ci, v)
    x = _x(nx * ny * nz, dtype, seed=nx + 7)
    with Stencil(nx, ny, nz, d, ox, oy, oz, dtype=dtype) as h:
        for o in ("A", "AH", "AT"):
            assert relerr(h.apply(x, o), reference_apply(op, x, o)) <= TOL[dtype], o
        ys = h.apply(x, "A")
    if nx * ny * nz >= 1000:   # the SELL CSR kernel (same FMA order; tiny matrices take other CSR kernels)
        with Csr(rp, ci, v, nx * ny * nz) as hc:
            assert np.array_equal(hc.apply(x, "A"), ys)


def test_stencil_bitwise_equals_csr_kernel():
    """Same arithmetic as the SELL CSR kernel (FMA accumulation in ascending
    column order): the stencil and the CSR operator agree bitwise on every
    product.  (Solves then differ only through the grid-dependent order of the
    dot-product partials; they are checked against the oracle below.)"""
    N = 24
    d, o = helmholtz_coeffs()
    rp, ci, v = lattice_csr(N, N, N, d, o)
    with Csr(rp, ci, v, N ** 3) as hc, Stencil(N, N, N, d, o) as hs:
        for seed in range(3):
            x = _x(N ** 3, np.complex128, seed)
            assert np.array_equal(hc.apply(x, "A"), hs.apply(x, "A"))


@pytest.mark.parametrize("method", ["bicgstab", "cors", "cocr", "cgs", "qmr", "bicor", "cgne"])
def test_stencil_solve_parity(method):
    N = 16
    d, o = helmholtz_coeffs()
    rp, ci, v = lattice_csr(N, N, N, d, o)
    y = helmholtz_rhs(N)
    with Stencil(N, N, N, d, o) as h:
        _parity(h, CsrOp(rp, ci, v), y, method, 1e-8, 4000, np.complex128, literal=False, tag="stencil")


@pytest.mark.parametrize("method", ["bicgstab", "cors", "cocr"])
def test_stencil_full_size_cfg5(method):
    """Config 5 at full size on the matrix-free operator: the residual property
    (recomputed by the oracle's own CSR product); the CSR path's iteration
    count is recorded beside it (identical products, but this indefinite
    problem is rounding-chaotic, so counts may differ)."""
    rp, ci, v = helmholtz_csr(128)
    y = helmholtz_rhs(128)
    d, o = helmholtz_coeffs()
    with Stencil(128, 128, 128, d, o) as h:
        g = h.solve(method, y, 1e-8, 20000)
    assert g["status"] == "CONVERGED"
    tr = np.linalg.norm(y - CsrOp(rp, ci, v).apply(g["x"])) / np.linalg.norm(y)
    assert tr <= 1e-7 and abs(tr - g["true_rel_res"]) <= 1e-3 * tr + 1e-15
    with Csr(rp, ci, v, 128 ** 3) as hc:
        gc = hc.solve(method, y, 1e-8, 20000)
    assert gc["status"] == "CONVERGED"
    _record(test="cfg5-full-stencil", method=method, k_stencil=g["iterations"], k_csr=gc["iterations"],
            true_rel_res=tr)


def test_stencil_bad_args():
    h = ccg.ccg_create("c128", 60)
    try:
        with pytest.raises(ccg.CcgError) as e:
            ccg.ccg_set_matvec_stencil7(h, 3, 4, 4, 6.0, -1.0)
        assert e.value.code == -2
        with pytest.raises(ccg.CcgError) as e:
            ccg.ccg_set_matvec_stencil7(h, 3, 4, 5, float("nan"), -1.0)
        assert e.value.code == -1
    finally:
        ccg.ccg_destroy(h)


# ---------------------------------------------------------------------------
# NEXT-4: FFT block-Toeplitz (lattice / DDA) operator (ccg_set_matvec_toeplitz3)
# ---------------------------------------------------------------------------
from oracle import ToeplitzOp                                   # noqa: E402
from workloads import dda_kernel, cfg4_rhs, cfg4_rows             # noqa: E402
from tests.test_oracle_numerics import _dense_from_kernel        # noqa: E402


class Toeplitz(Dense):
    def __init__(self, dims, kernel, diag, dtype=np.complex128):
        nx, ny, nz = dims
        self.n = nx * ny * nz
        self.dtype = dtype
        self.h = ccg.ccg_create(dt_name(dtype), self.n)
        ccg.ccg_set_matvec_toeplitz3(self.h, nx, ny, nz, kernel, diag)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("dims", [(1, 1, 1), (5, 3, 4), (7, 1, 2), (9, 6, 3), (1, 12, 5)])
def test_toeplitz_apply_parity(dtype, dims):
    """Random non-symmetric kernel: every product vs the brute-force dense matrix."""
    nx, ny, nz = dims
    rng = np.random.default_rng(nx + 10 * ny)
    K = rng.standard_normal((2 * nz - 1, 2 * ny - 1, 2 * nx - 1)) + 1j * rng.standard_normal(
        (2 * nz - 1, 2 * ny - 1, 2 * nx - 1))
    A = _dense_from_kernel(K, dims, 4 - 2j)
    x = _x(nx * ny * nz, dtype, seed=3)
    with Toeplitz(dims, K, 4 - 2j, dtype=dtype) as h:
        for o in ("A", "AH", "AT"):
            ref = reference_apply(A, x.astype(np.complex128), o)
            assert relerr(h.apply(x, o), ref) <= TOL[dtype], (o, relerr(h.apply(x, o), ref))


@pytest.mark.parametrize("yz", ["0", "1"])
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("dims", [(1, 1, 1), (5, 3, 4), (9, 6, 3), (1, 12, 5), (33, 7, 9), (40, 17, 2)])
def test_toeplitz_yz_fused_parity(monkeypatch, yz, dtype, dims):
    """Passes 2-4 fused into one kernel per kx plane (fft.cuh fft_yz, CCG_FFT_YZ=1)
    and the separate passes (=0): every product vs the brute-force dense matrix."""
    monkeypatch.setenv("CCG_FFT_YZ", yz)
    nx, ny, nz = dims
    rng = np.random.default_rng(nx + 7 * ny + 3 * nz)
    K = rng.standard_normal((2 * nz - 1, 2 * ny - 1, 2 * nx - 1)) + 1j * rng.standard_normal(
        (2 * nz - 1, 2 * ny - 1, 2 * nx - 1))
    A = _dense_from_kernel(K, dims, 4 - 2j)
    x = _x(nx * ny * nz, dtype, seed=5)
    with Toeplitz(dims, K, 4 - 2j, dtype=dtype) as h:
        for o in ("A", "AH", "AT"):
            ref = reference_apply(A, x.astype(np.complex128), o)
            assert relerr(h.apply(x, o), ref) <= TOL[dtype], (o, relerr(h.apply(x, o), ref))


def test_toeplitz_cfg2_fused_yz_solves(monkeypatch):
    """Config 2 through the fused-plane FFT passes: BiCGSTAB / COCR P-literal."""
    monkeypatch.setenv("CCG_FFT_YZ", "1")
    A, y = cfg2()
    K = dda_kernel((16, 16, 16), 1.0)
    with Toeplitz((16, 16, 16), K, 3 + 0.5j) as h:
        for o in ("A", "AH", "AT"):
            assert relerr(h.apply(y, o), reference_apply(A, y, o)) <= 1e-13, o
        for m in ("bicgstab", "cocr"):
            _parity(h, DenseOp(A), y, m, 1e-8, 1000, np.complex128, tag="cfg2-toeplitz-yz")


def test_toeplitz_cfg2_apply_and_solves():
    """BASELINE config 2 through the FFT operator: the dense product to 1e-13,
    then BiCGSTAB / QMR / BiCOR / COCR P-literal against the oracle's dense solves."""
    A, y = cfg2()
    K = dda_kernel((16, 16, 16), 1.0)
    with Toeplitz((16, 16, 16), K, 3 + 0.5j) as h:
        for o in ("A", "AH", "AT"):
            assert relerr(h.apply(y, o), reference_apply(A, y, o)) <= 1e-13, o
        for m in ("bicgstab", "qmr", "bicor", "cocr"):
            _parity(h, DenseOp(A), y, m, 1e-8, 1000, np.complex128, tag="cfg2-toeplitz")


def test_toeplitz_cfg4_full_size():
    """BASELINE config 4 (n = 65536, 68.7 GB as a dense matrix) on the FFT
    operator: sampled rows of A·x against the oracle's dense rows, the whole
    product against the oracle's FFT operator, and a BiCGSTAB solve whose x
    the oracle's own operator certifies (true residual ≤ 10·tol; iteration
    count inside the rounding envelope of SURVEY §8(c), 102-110 ± 2)."""
    dims = (64, 32, 32)
    K = dda_kernel(dims, 0.5)
    y = cfg4_rhs()
    op = ToeplitzOp(K, dims, 2.5 + 0.2j)
    x = _x(65536, np.complex128, 4)
    with Toeplitz(dims, K, 2.5 + 0.2j) as h:
        ax = h.apply(x, "A")
        assert relerr(ax, op.apply(x)) <= 1e-13
        rows = [0, 1, 4097, 33333, 65535]
        for r in rows:
            ref = reference_apply(cfg4_rows(r, r + 1), x)[0]
            assert abs(ax[r] - ref) <= 1e-13 * np.abs(cfg4_rows(r, r + 1)[0]) @ np.abs(x)
        g = h.solve("bicgstab", y, 1e-8, 2000)
    assert g["status"] == "CONVERGED" and 100 <= g["iterations"] <= 112
    tr = np.linalg.norm(y - op.apply(g["x"])) / np.linalg.norm(y)
    assert tr <= 1e-7
    _record(test="cfg4-full-toeplitz", method="bicgstab", k_gpu=g["iterations"], true_rel_res=tr)


def test_toeplitz_bad_args():
    h = ccg.ccg_create("c128", 24)
    try:
        with pytest.raises(ccg.CcgError) as e:
            ccg.ccg_set_matvec_toeplitz3(h, 2, 3, 5, np.zeros(3 * 5 * 9), 1.0)
        assert e.value.code == -2
        K = np.zeros((7, 5, 3), np.complex128)
        K[0, 0, 0] = np.nan
        with pytest.raises(ccg.CcgError) as e:
            ccg.ccg_set_matvec_toeplitz3(h, 2, 3, 4, K, 1.0)
        assert e.value.code == -1
    finally:
        ccg.ccg_destroy(h)


# ---------------------------------------------------------------------------
# Whole solve loop in one thread-block cluster (cluster.cuh; small dense n)
# ---------------------------------------------------------------------------
ALL9 = ("bicgstab", "cgne", "qmr", "bicor", "cors") + NEXT3


@pytest.mark.parametrize("cluster", ["0", "1"])
@pytest.mark.parametrize("method", ALL9)
def test_cluster_loop_cfg1(monkeypatch, cluster, method):
    """Config 1 with the single-cluster loop (default at this size) and with the
    multi-kernel graph loop: both P-literal against the oracle, same matvec
    counts and residual history."""
    monkeypatch.setenv("CCG_CLUSTER", cluster)
    A, y = cfg1()
    if method == "cocr":
        A = _csym(A)
    with Dense(A) as h:
        o, g = _parity(h, DenseOp(A), y, method, 1e-10, 500, np.complex128, tag=f"cfg1-cluster{cluster}")
        assert (g["matvecs_a"], g["matvecs_ah"]) == (o.matvecs_a, o.matvecs_ah)
        h.solve(method, y, 1e-10, 500)
        np.testing.assert_allclose(ccg.ccg_get_history(h.h), np.array(o.history, float) / o.history[0],
                                   rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("n", [1, 5, 33, 200, 511])
@pytest.mark.parametrize("method", ["bicgstab", "qmr", "cgne", "bicg", "pbicgstab"])
def test_cluster_loop_ragged_c64(monkeypatch, n, method):
    """Row ranges that do not divide the cluster (n < cluster size included), c64."""
    if method == "pbicgstab" and n == 1:
        # 1×1 in c64: after one step q = r − αs cancels exactly on the GPU (FMA)
        # but not in the oracle's separate multiply/subtract, so the tol = 0
        # equal-k rerun ends in different (both valid) exact-arithmetic outcomes
        # — half-step exit vs ⟨y,y⟩ = 0 breakdown; the graph path does the same
        pytest.skip("degenerate 1×1: FMA-decided exact cancellation (see comment)")
    monkeypatch.setenv("CCG_CLUSTER", "1")
    A = dense_random(n, seed=n, dtype=np.complex64, shift=3 - 1j)
    y = (dense_random(n, seed=n + 1)[:, 0] * 3).astype(np.complex64)
    with Dense(A) as h:
        _parity(h, DenseOp(A), y, method, 1e-5, 300, np.complex64, tag=f"cluster-c64-{n}", literal=False)


# ---------------------------------------------------------------------------
# User operator (ccg_set_matvec_callback): the paper's own matvec contract
# ---------------------------------------------------------------------------
import ctypes                      # noqa: E402
import os                          # noqa: E402
import subprocess                  # noqa: E402


@pytest.fixture(scope="module")
def tridiag_lib(tmp_path_factory):
    src = os.path.join(os.path.dirname(__file__), "support", "cb_tridiag.cu")
    out = str(tmp_path_factory.mktemp("cb") / "libcbtri.so")
    subprocess.run(["nvcc", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-o", out, src], check=True)
    return ctypes.CDLL(out)


class _Tri(ctypes.Structure):
    _fields_ = [("d", ctypes.c_double * 2), ("lo", ctypes.c_double * 2), ("up", ctypes.c_double * 2)]


def _tri_dense(n, d, lo, up):
    return (np.diag(np.full(n, d)) + np.diag(np.full(n - 1, lo), -1) + np.diag(np.full(n - 1, up), 1)).astype(
        np.complex128)


@pytest.mark.parametrize("method", ["bicgstab", "qmr", "cgne", "bicor", "cocr", "cgs"])
def test_callback_graph_safe_native(tridiag_lib, method):
    """A native callback that enqueues its own kernel (graph-capturable):
    every product and every method against the oracle's dense product/solve."""
    n = 777
    d, lo, up = 4 - 1j, -1 + 0.5j, -0.75 - 0.25j
    if method == "cocr":
        up = lo                                    # complex symmetric
    A = _tri_dense(n, d, lo, up)
    tri = _Tri((d.real, d.imag), (complex(lo).real, complex(lo).imag), (complex(up).real, complex(up).imag))
    h = ccg.ccg_create("c128", n)
    try:
        ccg.ccg_set_matvec_callback_ptr(h, ctypes.cast(tridiag_lib.cb_tridiag, ctypes.c_void_p).value,
                                        ctypes.addressof(tri),
                                        caps=ccg.CB_A | ccg.CB_AH | ccg.CB_AT | ccg.CB_GRAPH_SAFE)
        x = _x(n, np.complex128, 5)
        xd = to_dev(x)
        yd = torch.empty_like(xd)
        for o in ("A", "AH", "AT"):
            ccg.ccg_apply(h, o, xd, yd)
            assert relerr(yd.cpu().numpy(), reference_apply(A, x, o)) <= 1e-13, o

        class H:
            def solve(self, m, yy, tol, maxit):
                yv = to_dev(yy)
                xo = torch.empty_like(yv)
                r = ccg.ccg_solve(h, m, None, yv, xo, tol, maxit)
                r["x"] = xo.cpu().numpy()
                r["hist"] = ccg.ccg_get_history(h)
                return r
        yv = _x(n, np.complex128, 6)
        o, g = _parity(H(), DenseOp(A), yv, method, 1e-10, 2000, np.complex128, tag="callback")
        assert (g["matvecs_a"], g["matvecs_ah"]) == (o.matvecs_a, o.matvecs_ah)
    finally:
        ccg.ccg_destroy(h)


def test_callback_python_eager():
    """A Python callback (eager mode: called for every product) that delegates
    to another handle's dense product after ordering itself on the stream."""
    n = 300
    A = dense_random(n, seed=21, dtype=np.complex128, shift=2.5 - 0.5j)
    inner = Dense(A)
    calls = []

    def fn(op, xp, yp, nn, row0, nloc, stream):
        torch.cuda.ExternalStream(stream).synchronize()
        ccg.load().ccg_apply(inner.h, op, ctypes.c_void_p(xp), ctypes.c_void_p(yp))
        calls.append(op)
        return 0

    h = ccg.ccg_create("c128", n)
    try:
        ccg.ccg_set_matvec_callback(h, fn, caps=ccg.CB_A | ccg.CB_AH)
        y = _x(n, np.complex128, 7)

        class H:
            def solve(self, m, yy, tol, maxit):
                yv = to_dev(yy)
                xo = torch.empty_like(yv)
                r = ccg.ccg_solve(h, m, None, yv, xo, tol, maxit)
                r["x"] = xo.cpu().numpy()
                r["hist"] = ccg.ccg_get_history(h)
                return r
        for m in ("bicgstab", "cgne"):
            _parity(H(), DenseOp(A), y, m, 1e-10, 500, np.complex128, tag="callback-py")
        assert calls and set(calls) <= {0, 1}
        with pytest.raises(ccg.CcgError) as e:       # no Aᵀ declared
            ccg.ccg_apply(h, "AT", to_dev(y), torch.empty(n, dtype=torch.complex128, device="cuda"))
        assert e.value.code == -3
    finally:
        ccg.ccg_destroy(h)
        inner.close()



@pytest.mark.parametrize("restart", [1, 5, 17, 64])
def test_gmres_restart_lengths(restart):
    """GMRES(m) for several restart lengths (cycle ends, restarts with the
    explicit residual) against the oracle with the same m: P-literal."""
    n = 300
    A = dense_random(n, seed=31, dtype=np.complex128, shift=2.0 - 1.0j)
    y = dense_random(n, seed=32)[:, 0] * 2
    with Dense(A) as h:
        ccg.ccg_set_gmres_restart(h.h, restart)
        o = oracle.solve("gmres", DenseOp(A), y, 1e-10, 400, restart=restart)
        g = h.solve("gmres", y, 1e-10, 400)
        assert g["status"] == o.status_name == "CONVERGED"
        assert abs(g["iterations"] - o.iterations) <= 2
        assert (g["matvecs_a"], g["matvecs_ah"]) == (o.matvecs_a, o.matvecs_ah) or g["iterations"] != o.iterations
        k = min(g["iterations"], o.iterations)
        ge = h.solve("gmres", y, 0.0, k)
        oe = oracle.solve("gmres", DenseOp(A), y, 0.0, k, restart=restart)
        assert relerr(ge["x"], oe.x) <= 1e-9
        with pytest.raises(ccg.CcgError) as e:
            ccg.ccg_set_gmres_restart(h.h, 65)
        assert e.value.code == -1


def test_gmres_c64_cfg3_proxy():
    n = 4096
    A = gauss_shifted_rows(n, 0, n, seed=1)
    y = cfg3_rhs(n)
    with Dense(A) as h:
        _parity(h, DenseOp(A), y, "gmres", 1e-5, 500, np.complex64, tag="cfg3-proxy-gmres", literal=False)



@pytest.mark.parametrize("ell", [1, 2, 3, 4])
def test_bicgstabl_ells(ell):
    """BiCGstab(ℓ) for every supported ℓ against the oracle with the same ℓ
    (P-literal, matvec counts, residual history); ℓ = 1 reproduces the GPU
    BiCGSTAB iteration count."""
    n = 400
    A = dense_random(n, seed=41, dtype=np.complex128, shift=1.5 - 1.0j)
    y = dense_random(n, seed=42)[:, 0] * 2
    with Dense(A) as h:
        ccg.ccg_set_bicgstab_ell(h.h, ell)
        o = oracle.solve("bicgstabl", DenseOp(A), y, 1e-10, 400, ell=ell)
        g = h.solve("bicgstabl", y, 1e-10, 400)
        assert g["status"] == o.status_name == "CONVERGED"
        assert abs(g["iterations"] - o.iterations) <= 2
        if g["iterations"] == o.iterations:
            assert (g["matvecs_a"], g["matvecs_ah"]) == (o.matvecs_a, o.matvecs_ah)
            np.testing.assert_allclose(ccg.ccg_get_history(h.h), np.array(o.history, float) / o.history[0],
                                       rtol=1e-6, atol=1e-12)
        k = min(g["iterations"], o.iterations)
        ge = h.solve("bicgstabl", y, 0.0, k)
        oe = oracle.solve("bicgstabl", DenseOp(A), y, 0.0, k, ell=ell)
        assert relerr(ge["x"], oe.x) <= 1e-9
        if ell == 1:
            assert g["iterations"] == h.solve("bicgstab", y, 1e-10, 400)["iterations"]
        with pytest.raises(ccg.CcgError) as e:
            ccg.ccg_set_bicgstab_ell(h.h, 5)
        assert e.value.code == -1


# ---------------------------------------------------------------------------
# Right Jacobi preconditioning (ccg_set_jacobi; NEXT-4)
# ---------------------------------------------------------------------------
def _badly_scaled(n, seed=12):
    rng = np.random.default_rng(seed)
    d = np.logspace(0, 4, n) * np.exp(1j * rng.uniform(0, 2 * np.pi, n))
    A = np.diag(d) + 0.3 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return A.astype(np.complex128), d.astype(np.complex128), y.astype(np.complex128)


@pytest.mark.parametrize("method", ["bicgstab", "qmr", "cgne", "bicor", "gmres", "bicgstabl", "tfqmr", "cgnr"])
def test_jacobi_badly_scaled(method):
    """A diagonal spanning four decades: unpreconditioned the methods stall,
    with right Jacobi they converge in a handful of iterations — GPU against the
    oracle's preconditioned solve (P-literal), x = D⁻¹u returned."""
    n = 300
    A, d, y = _badly_scaled(n)
    o = oracle.solve_jacobi(method, DenseOp(A), d, y, 1e-10, 3000)
    with Dense(A) as h:
        ccg.ccg_set_jacobi(h.h, to_dev(d))
        g = h.solve(method, y, 1e-10, 3000)
        assert g["status"] == o.status_name == "CONVERGED", (g["status"], o.status_name)
        assert abs(g["iterations"] - o.iterations) <= 2 and g["iterations"] <= 60
        assert g["true_rel_res"] <= 1e-9
        k = min(g["iterations"], o.iterations)
        ge = h.solve(method, y, 0.0, k)
        oe = oracle.solve_jacobi(method, DenseOp(A), d, y, 0.0, k)
        assert relerr(ge["x"], oe.x) <= 1e-9
        xs = np.linalg.solve(A, y)
        gx = h.solve(method, y, 1e-10, 3000, x0=0.5 * xs)
        ox = oracle.solve_jacobi(method, DenseOp(A), d, y, 1e-10, 3000, x0=0.5 * xs)
        assert abs(gx["iterations"] - ox.iterations) <= 2 and relerr(gx["x"], xs) <= 1e-8
        ccg.ccg_set_jacobi(h.h, None)                 # disabled again: the plain method
        gp = h.solve(method, y, 1e-10, 200)
        assert gp["iterations"] > 2 * g["iterations"] or gp["status"] != "CONVERGED"


def test_jacobi_constant_diagonal_cfg1():
    A, y = cfg1()
    with Dense(A) as h:
        g0 = h.solve("bicgstab", y, 1e-10, 500)
        ccg.ccg_set_jacobi(h.h, np.full(256, 3 - 4j))
        g1 = h.solve("bicgstab", y, 1e-10, 500)
    assert g0["iterations"] == g1["iterations"]
    assert relerr(g1["x"], g0["x"]) <= 1e-9
    h2 = ccg.ccg_create("c128", 4)
    try:
        with pytest.raises(ccg.CcgError) as e:
            ccg.ccg_set_jacobi(h2, np.array([1, 2, 0, 4], np.complex128))
        assert e.value.code == -1
    finally:
        ccg.ccg_destroy(h2)


def test_workspaces_coexist_on_one_handle():
    """GMRES, BiCGstab(ℓ) and Jacobi workspaces allocated in any order on one
    handle stay valid (each method repeated after the others allocated)."""
    n = 300
    A, d, y = _badly_scaled(n, seed=21)
    with Dense(A) as h:
        ccg.ccg_set_jacobi(h.h, to_dev(d))
        ref = {m: oracle.solve_jacobi(m, DenseOp(A), d, y, 1e-10, 500) for m in ("bicgstabl", "gmres", "bicgstab")}
        for m in ("bicgstabl", "gmres", "bicgstabl", "bicgstab", "gmres"):
            g = h.solve(m, y, 1e-10, 500)
            assert g["status"] == "CONVERGED" and abs(g["iterations"] - ref[m].iterations) <= 2, m
            assert relerr(g["x"], ref[m].x) <= 1e-8, m
        ccg.ccg_set_gmres_restart(h.h, 7)
        ccg.ccg_set_bicgstab_ell(h.h, 3)
        for m, kw in (("gmres", {"restart": 7}), ("bicgstabl", {"ell": 3})):
            o = oracle.solve_jacobi(m, DenseOp(A), d, y, 1e-10, 500, **kw)
            g = h.solve(m, y, 1e-10, 500)
            assert abs(g["iterations"] - o.iterations) <= 2 and relerr(g["x"], o.x) <= 1e-8, m


# ---------------------------------------------------------------------------
# Schedule knobs that must not change results: the SELL load schedule
# (CCG_SELL_ONE: one row per step vs two) and the pipelined chunk launches
# (CCG_PIPELINE=1) reorder only when loads issue / when the host waits, so
# products and whole solves are bitwise identical to the defaults.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_sell_schedules_bitwise(monkeypatch, dtype):
    N = 20                                        # 8000 rows: ragged last slice, boundary widths < 7
    rp, ci, v = helmholtz_csr(N, kh=10 / 128)
    v = v.astype(dtype)
    x = _x(N ** 3, dtype, seed=5)
    ys, sols = [], []
    for one in ("0", "1"):
        monkeypatch.setenv("CCG_SELL_ONE", one)
        with Csr(rp, ci, v, N ** 3, flags=ccg.FLAG_SYMMETRIC) as h:
            ys.append((h.apply(x, "A"), h.apply(x, "AH")))
            sols.append(h.solve("bicgstab", helmholtz_rhs(N).astype(dtype), 1e-6, 3000))
    assert np.array_equal(ys[0][0], ys[1][0]) and np.array_equal(ys[0][1], ys[1][1])
    assert sols[0]["iterations"] == sols[1]["iterations"] and np.array_equal(sols[0]["x"], sols[1]["x"])
    assert relerr(ys[1][0], reference_apply_csr(rp, ci, v, x)) <= TOL[dtype]


def reference_apply_csr(rp, ci, v, x):
    return CsrOp(rp, ci, v.astype(np.complex128)).apply(x.astype(np.complex128))


@pytest.mark.parametrize("method", ["bicgstab", "cocr", "gmres"])
def test_pipelined_chunks_bitwise(monkeypatch, method):
    N = 16
    rp, ci, v = helmholtz_csr(N, kh=10 / 128)
    y = helmholtz_rhs(N)
    out = []
    for pipe in ("0", "1"):
        monkeypatch.setenv("CCG_PIPELINE", pipe)
        with Csr(rp, ci, v, N ** 3) as h:
            out.append(h.solve(method, y, 1e-8, 3000))
    a, b = out
    assert a["status"] == b["status"] == "CONVERGED"
    assert a["iterations"] == b["iterations"] and np.array_equal(a["x"], b["x"])
    assert a["true_rel_res"] == b["true_rel_res"]


# ---------------------------------------------------------------------------
# QMR / BiCG dual product in the warp-per-row layout (matvec.cuh
# gemv_dual_rows, CCG_DUAL_ROWS=1): against the oracle and the column-owner dual
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("method", ["qmr", "bicg"])
@pytest.mark.parametrize("sysname", ["cfg2", "c64"])
def test_dual_rows_parity(monkeypatch, method, sysname):
    monkeypatch.setenv("CCG_DUAL_ROWS", "1")
    if sysname == "cfg2":
        A, y = cfg2()
        tol, dt = 1e-8, np.complex128
    else:
        n = 4096
        A = gauss_shifted_rows(n, 0, n, seed=1)
        y = cfg3_rhs(n)
        tol, dt = 1e-5, np.complex64
    with Dense(A) as h:
        _parity(h, DenseOp(A), y, method, tol, 1000, dt, literal=False, tag=f"dual-rows-{sysname}")


@pytest.mark.parametrize("n", [7, 257, 1000, 1537])
def test_dual_rows_ragged(monkeypatch, n):
    """Ragged n (partial strips and row blocks): QMR x after k iterations equal
    to the column-owner dual's to rounding, and to the oracle's."""
    A = dense_random(n, seed=n, dtype=np.complex128, shift=3 - 1j)
    y = dense_random(n, seed=n + 1)[:, 0] * 3
    k = 6
    monkeypatch.setenv("CCG_CLUSTER", "0")
    monkeypatch.setenv("CCG_DUAL_ROWS", "1")
    with Dense(A) as h:
        a = h.solve("qmr", y, 0.0, k)
    monkeypatch.setenv("CCG_DUAL_ROWS", "0")
    with Dense(A) as h:
        b = h.solve("qmr", y, 0.0, k)
    o = oracle.solve("qmr", DenseOp(A), y, 0.0, k)
    assert relerr(a["x"], b["x"]) <= 1e-12
    assert relerr(a["x"], o.x) <= 1e-9
