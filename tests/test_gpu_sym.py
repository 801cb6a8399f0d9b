"""Complex-symmetric dense operator read from its upper triangle
(CCG_FLAG_SYMMETRIC on ccg_set_matvec_dense, one rank; matvec.cuh gemv_sym).

The DDA matrices the paper's methods target are complex symmetric, A = Aᵀ
(§1, DDSCAT; the COCR/BiCOR/CORS family of P:69 §2.4 and P:87 §3.4
is built for them; BASELINE configs 2 and 4 are bitwise symmetric, SURVEY
§8(d)).  With the flag the library reads only j ≥ i:
    y_i = Σ_{j ≥ i} A_ij x_j + Σ_{j < i} A_ji x_j,
half of A's bytes per product.  The product is the same matrix-vector product
in another summation order, so it is held to the per-matvec bar against the
oracle's full product (1e-13 c128 / 1e-5 c64 normwise), and
solves to the same bars as the full-matrix path.
"""

import numpy as np
import pytest

import oracle
from oracle import DenseOp
from oracle.operators import reference_apply
import paper_1208_4869_b200 as ccg
from tests._gpu import Dense, TOL, relerr
from tests.test_gpu_solve import _parity
from workloads import cfg2, dense_random

pytestmark = pytest.mark.gpu


def _sym(n, dtype, seed):
    G = dense_random(n, seed=seed, dtype=np.complex128, shift=3 - 1j)
    A = 0.5 * (G + G.T)
    A = np.triu(A) + np.triu(A, 1).T          # bitwise A = Aᵀ
    assert np.array_equal(A, A.T)
    return A.astype(dtype)


def _x(n, dtype, seed):
    rng = np.random.default_rng(seed)
    return ((rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2)).astype(dtype)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("n", [1, 2, 7, 255, 256, 257, 511, 1000, 1537, 4096])
def test_sym_apply_parity(dtype, n):
    if dtype == np.complex64 and n % 2:
        n += 1                               # c64 needs even n for the vectorised layout
    A = _sym(n, dtype, seed=n)
    x = _x(n, dtype, seed=n + 1)
    with Dense(A, flags=ccg.FLAG_SYMMETRIC) as h:
        for op in ("A", "AH", "AT"):
            got = h.apply(x, op)
            ref = reference_apply(A.astype(np.complex128), x.astype(np.complex128), op)
            assert relerr(got, ref) <= TOL[dtype], (op, relerr(got, ref))
            # componentwise: every row sums the same terms as the full product
            den = np.abs(A).astype(np.float64) @ np.abs(x).astype(np.float64)
            eps = np.finfo(np.float64 if dtype == np.complex128 else np.float32).eps
            assert np.all(np.abs(got - ref) <= 4 * n * eps * den + 1e-300), op


@pytest.mark.parametrize("H", ["8", "32", "512"])
def test_sym_tile_heights(monkeypatch, H):
    """Every row-block height (CCG_SYM_H) tiles the triangle exactly once."""
    monkeypatch.setenv("CCG_SYM_H", H)
    n = 777
    A = _sym(n, np.complex128, seed=3)
    x = _x(n, np.complex128, seed=4)
    with Dense(A, flags=ccg.FLAG_SYMMETRIC) as h:
        assert relerr(h.apply(x), reference_apply(A, x, "A")) <= TOL[np.complex128]


def test_sym_bitwise_repeatable():
    A, y = cfg2()
    with Dense(A, flags=ccg.FLAG_SYMMETRIC) as h:
        a = h.apply(y)
        b = h.apply(y)
        assert np.array_equal(a, b)
        s1 = h.solve("bicgstab", y, 1e-8, 1000)
        s2 = h.solve("bicgstab", y, 1e-8, 1000)
        assert np.array_equal(s1["x"], s2["x"]) and s1["iterations"] == s2["iterations"]


def test_sym_reads_upper_triangle_only():
    """The strictly-lower triangle is never read: poisoning it with NaN leaves
    the product finite and equal to the symmetric product."""
    n = 1000
    A = _sym(n, np.complex128, seed=11)
    P = A.copy()
    P[np.tril_indices(n, -1)] = np.nan
    x = _x(n, np.complex128, seed=12)
    with Dense(P, flags=ccg.FLAG_SYMMETRIC) as h:
        for op in ("A", "AH", "AT"):
            assert relerr(h.apply(x, op), reference_apply(A, x, op)) <= TOL[np.complex128], op


@pytest.mark.parametrize("method", ["bicgstab", "cgne", "qmr", "bicor", "cors", "cocr"])
def test_sym_cfg2_solve_parity(method):
    """BASELINE config 2 (dense c128 n = 4096, A = Aᵀ) through the upper-
    triangle products: the same bars as test_gpu_solve.test_cfg2_all_methods
    (P-literal where that test is literal, else the P-envelope)."""
    A, y = cfg2()
    with Dense(A, flags=ccg.FLAG_SYMMETRIC) as h:
        _parity(h, DenseOp(A), y, method, 1e-8, 1000, np.complex128, tag="cfg2-sym",
                literal=method in ("bicgstab", "qmr", "bicor"))


@pytest.mark.parametrize("method", ["bicgstab", "cors", "qmr"])
def test_sym_c64_solve_parity(method):
    n = 2048
    A = _sym(n, np.complex64, seed=21)
    y = _x(n, np.complex64, seed=22)
    with Dense(A, flags=ccg.FLAG_SYMMETRIC) as h:
        _parity(h, DenseOp(A), y, method, 1e-5, 500, np.complex64, tag="sym-c64", literal=False)


def test_sym_off_matches_full(monkeypatch):
    """CCG_SYMV=0 with the flag reads all of A (the general kernels): the two
    products agree to the per-matvec bar."""
    A, y = cfg2()
    with Dense(A, flags=ccg.FLAG_SYMMETRIC) as hs:
        ys = hs.apply(y)
    monkeypatch.setenv("CCG_SYMV", "0")
    with Dense(A, flags=ccg.FLAG_SYMMETRIC) as hf:
        yf = hf.apply(y)
    assert relerr(ys, yf) <= TOL[np.complex128]


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_sym_dual_qmr(monkeypatch, dtype):
    """QMR's A·p and Aᴴ·q from one upper-triangle pass (gemv_sym_dual) against
    the same iteration with two single symmetric products (CCG_QMR_DUAL=0):
    rounding-level agreement at equal k, and both against the oracle."""
    n = 1536 if dtype == np.complex128 else 2048
    A = _sym(n, dtype, seed=31)
    y = _x(n, dtype, seed=32)
    k = 12
    with Dense(A, flags=ccg.FLAG_SYMMETRIC) as h:
        a = h.solve("qmr", y, 0.0, k)
    monkeypatch.setenv("CCG_QMR_DUAL", "0")
    with Dense(A, flags=ccg.FLAG_SYMMETRIC) as h:
        b = h.solve("qmr", y, 0.0, k)
    o = oracle.solve("qmr", DenseOp(A), y, 0.0, k)
    bar = 1e-12 if dtype == np.complex128 else 1e-4
    assert relerr(a["x"], b["x"]) <= bar
    assert relerr(a["x"], o.x) <= (1e-9 if dtype == np.complex128 else 1e-4)


def test_sym_detected_without_flag(monkeypatch):
    """Without CCG_FLAG_SYMMETRIC a bitwise-symmetric A is detected on the
    device (CCG_STAT_SYMMETRIC = 2) and takes the upper-triangle products; one
    changed element (or CCG_SYM_DETECT=0) keeps the general path (0)."""
    monkeypatch.setenv("CCG_SYM_DETECT", "1")   # the library default (conftest pins 0)
    A, y = cfg2()
    with Dense(A) as h:
        assert ccg.ccg_get_stat(h.h, "symmetric") == 2
        assert relerr(h.apply(y), reference_apply(A, y, "A")) <= TOL[np.complex128]
        _parity(h, DenseOp(A), y, "bicgstab", 1e-8, 1000, np.complex128, tag="cfg2-sym-detected")
    with Dense(A, flags=ccg.FLAG_SYMMETRIC) as h:
        assert ccg.ccg_get_stat(h.h, "symmetric") == 1
    for (i, j) in ((4095, 0), (0, 4095), (2000, 2001), (17, 3)):
        B = A.copy()
        B[i, j] += 1e-3
        with Dense(B) as h:
            assert ccg.ccg_get_stat(h.h, "symmetric") == 0, (i, j)
            assert relerr(h.apply(y), reference_apply(B, y, "A")) <= TOL[np.complex128]
    monkeypatch.setenv("CCG_SYM_DETECT", "0")
    with Dense(A) as h:
        assert ccg.ccg_get_stat(h.h, "symmetric") == 0


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("n", [1, 2, 31, 33, 100, 1000])
def test_sym_detect_ragged(monkeypatch, dtype, n):
    """Ragged n (partial 32×32 tiles): symmetric detected, a single flipped
    entry anywhere in the last partial tile row is not; products exact."""
    monkeypatch.setenv("CCG_SYM_DETECT", "1")
    if dtype == np.complex64 and n % 2:
        n += 1
    A = _sym(n, dtype, seed=40 + n)
    x = _x(n, dtype, seed=41)
    with Dense(A) as h:
        assert ccg.ccg_get_stat(h.h, "symmetric") == 2
        assert relerr(h.apply(x), reference_apply(A.astype(np.complex128), x.astype(np.complex128), "A")) \
            <= TOL[dtype]
    if n > 1:
        B = A.copy()
        j = (n - 1) // 2                       # off the diagonal (j < n − 1)
        B[n - 1, j] = B[n - 1, j] * (1 + 1e-3)
        with Dense(B) as h:
            assert ccg.ccg_get_stat(h.h, "symmetric") == 0


@pytest.mark.parametrize("k", [1, 2, 7, 20])
def test_sym_bs_fuse_bitwise(monkeypatch, k):
    """BiCGSTAB's P and S passes folded into the upper-triangle product (x
    staged through BsPIn / BsSIn, the stage-2 epilogue stores p / s): the same
    recurrence bit for bit as the separate passes (CCG_BS_FUSE=0)."""
    A, y = cfg2()
    res = []
    for f in ("0", "1"):
        monkeypatch.setenv("CCG_BS_FUSE", f)
        with Dense(A, flags=ccg.FLAG_SYMMETRIC) as h:
            res.append(h.solve("bicgstab", y, 0.0, k))
    a, b = res
    assert a["iterations"] == b["iterations"] == k
    assert np.array_equal(a["x"], b["x"])
    assert np.array_equal(np.asarray(a["hist"]), np.asarray(b["hist"]))
