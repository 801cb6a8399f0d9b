"""Pins for oracle.solvers (CPU only).

The recurrences cannot be checked against a library routine (none exists for
these methods), so each is pinned by what the mathematics fixes
(SURVEY.md §8(c) pin table):

* exact Gaussian-rational arithmetic: finite termination at iteration n with
  A·x == y exactly (CGNE, BiCOR, CORS; BiCGSTAB at the half-step of n);
* 100-digit mpmath: QMR terminates at iteration n;
* textbook reductions: QMR ≡ MINRES on Hermitian A (dense least squares over
  the Krylov space), BiCOR ≡ BiCG(shadow Aᴴr₀*), CORS ≡ CGS(shadow Aᴴr₀*),
  BiCOR(r₀* = conj r₀) ≡ COCR on complex-symmetric A, QMR Aᴴ-form ≡ Aᵀ-form;
* special cases: A = cI converges in one iteration to y/c; unitary A → CGNE
  in one iteration; CGNE error is monotone;
* the dense LU solution (oracle.direct) at n ≤ 64; true vs recurrence
  residual; scale invariance; work accounting; breakdown / non-finite /
  zero-rhs handling.

A plausible slip in any recurrence (dropped term, wrong conjugation, wrong
sign or index) breaks finite termination or one of the equivalences.
"""

import numpy as np
import pytest

from oracle import solve, DenseOp
from oracle.solvers import CONVERGED, MAXIT, BREAKDOWN, NONFINITE, HOT_PATH
from oracle.exact import to_exact
from oracle.direct import lu_solve
from workloads import dense_random, cfg1

RATIONAL = ("bicgstab", "cgne", "bicor", "cors")


def _rand_int(n, seed, herm_pd=False):
    rng = np.random.default_rng(seed)
    A = rng.integers(-4, 5, (n, n)) + 1j * rng.integers(-4, 5, (n, n))
    if herm_pd:
        A = A @ A.conj().T + np.eye(n)
    else:
        A = A + 6 * np.eye(n)
    y = rng.integers(-3, 4, n) + 1j * rng.integers(-3, 4, n)
    return A.astype(np.complex128), y.astype(np.complex128)


# ---------------- special cases ----------------
@pytest.mark.parametrize("method", HOT_PATH)
def test_scaled_identity_one_iteration(method):
    c = 3 - 4j
    n = 10
    rng = np.random.default_rng(0)
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    res = solve(method, DenseOp(c * np.eye(n, dtype=np.complex128)), y, 1e-12, 50)
    assert res.status == CONVERGED and res.iterations == 1
    np.testing.assert_allclose(res.x, y / c, rtol=1e-15, atol=1e-15)
    if method == "bicgstab":
        assert res.half_step and res.matvecs_a == 1


@pytest.mark.parametrize("method", HOT_PATH)
def test_identity_spec_example(method):
    """S:314 / S:323 / S:341: identity → ≤ 1 iteration, x̂ == y."""
    y = np.arange(5) + 2j
    res = solve(method, DenseOp(np.eye(5, dtype=np.complex128)), y, 1e-10, 10)
    assert res.status == CONVERGED and res.iterations <= 1
    np.testing.assert_allclose(res.x, y, rtol=1e-15)


def test_cgne_unitary_one_iteration():
    n = 4
    F = np.exp(-2j * np.pi * np.outer(np.arange(n), np.arange(n)) / n) / np.sqrt(n)
    y = np.array([1, 2j, -1, 0.5])
    res = solve("cgne", DenseOp(F), y, 1e-12, 10)
    assert res.status == CONVERGED and res.iterations == 1


# ---------------- exact arithmetic: finite termination ----------------
@pytest.mark.parametrize("n", [3, 4, 5, 6])
@pytest.mark.parametrize("herm_pd", [False, True])
@pytest.mark.parametrize("method", RATIONAL)
def test_exact_finite_termination(method, n, herm_pd):
    A, y = _rand_int(n, seed=10 * n + herm_pd, herm_pd=herm_pd)
    Ae, ye = to_exact(A), to_exact(y)
    op = DenseOp(Ae)
    res = solve(method, op, ye, 0.0, n + 3)
    assert res.status == CONVERGED, (res.status_name, res.breakdown)
    assert res.iterations <= n
    r = ye - op.apply(res.x)
    assert all(v == 0 for v in r), "A·x must equal y exactly"
    if not herm_pd:
        # generic nonsymmetric A: termination exactly at n, not before
        assert res.iterations == n
        if method == "bicgstab":
            assert res.half_step and res.matvecs_a == 2 * n - 1


@pytest.mark.parametrize("n", [4, 6])
def test_qmr_mpmath_termination(n):
    mpmath = pytest.importorskip("mpmath")
    A, y = _rand_int(n, seed=100 + n)
    with mpmath.workdps(100):
        Am = np.array([[mpmath.mpc(complex(v)) for v in row] for row in A], dtype=object)
        ym = np.array([mpmath.mpc(complex(v)) for v in y], dtype=object)
        res = solve("qmr", DenseOp(Am), ym, 1e-90, n + 2)
        assert res.status == CONVERGED and res.iterations == n
        r = ym - Am.dot(res.x)
        rel = mpmath.sqrt(sum(abs(v) ** 2 for v in r)) / mpmath.sqrt(sum(abs(v) ** 2 for v in ym))
        assert rel < mpmath.mpf("1e-90")


# ---------------- textbook reductions ----------------
@pytest.mark.parametrize("definite", [True, False])
def test_qmr_is_minres_on_hermitian(definite):
    n = 40
    rng = np.random.default_rng(7)
    B = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    H = (B + B.conj().T) / 2
    A = H + (12 * np.eye(n) if definite else 0.3 * np.eye(n))
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for k in range(1, 9):
        res = solve("qmr", DenseOp(A), y, 0.0, k)
        assert res.iterations == k
        K = np.empty((n, k), dtype=np.complex128)
        K[:, 0] = y
        for j in range(1, k):
            K[:, j] = A @ K[:, j - 1]
        Q, _ = np.linalg.qr(K)
        c, *_ = np.linalg.lstsq(A @ Q, y, rcond=None)
        xm = Q @ c
        assert np.linalg.norm(res.x - xm) <= 1e-10 * np.linalg.norm(xm)


def test_qmr_hermitian_and_transpose_forms_agree():
    A = dense_random(30, seed=21, shift=2.0)
    y = dense_random(30, seed=22)[:, 0] * 5
    rh = solve("qmr", DenseOp(A), y, 1e-12, 200, form="H")
    rt = solve("qmr", DenseOp(A), y, 1e-12, 200, form="T")
    assert rh.iterations == rt.iterations and rh.status == CONVERGED
    np.testing.assert_allclose(rh.history, rt.history, rtol=1e-10, atol=1e-13 * rh.history[0])
    assert np.linalg.norm(rh.x - rt.x) <= 1e-13 * np.linalg.norm(rh.x)


@pytest.mark.parametrize("shadow", ["r0", "Ar0", "conj"])
def test_bicor_is_bicg_with_ah_shadow(shadow):
    A = dense_random(24, seed=31, shift=2 + 1j)
    y = dense_random(24, seed=32)[:, 1] * 4
    rs = {"r0": y, "Ar0": A @ y, "conj": np.conj(y)}[shadow]
    a = solve("bicor", DenseOp(A), y, 1e-12, 100, shadow=rs)
    b = solve("bicg", DenseOp(A), y, 1e-12, 100, shadow=A.conj().T @ rs)
    assert a.iterations == b.iterations and a.status == CONVERGED
    np.testing.assert_allclose(a.history, b.history, rtol=1e-9, atol=1e-13 * a.history[0])
    assert np.linalg.norm(a.x - b.x) <= 1e-12 * np.linalg.norm(a.x)


def test_cors_is_cgs_with_ah_shadow():
    A = dense_random(24, seed=41, shift=2 + 1j)
    y = dense_random(24, seed=42)[:, 1] * 4
    a = solve("cors", DenseOp(A), y, 1e-12, 100)
    b = solve("cgs", DenseOp(A), y, 1e-12, 100, shadow=A.conj().T @ y)
    assert a.iterations == b.iterations and a.status == CONVERGED
    np.testing.assert_allclose(a.history, b.history, rtol=1e-8, atol=1e-13 * a.history[0])
    assert np.linalg.norm(a.x - b.x) <= 1e-11 * np.linalg.norm(a.x)


def test_bicor_conj_shadow_is_cocr_on_complex_symmetric():
    B = dense_random(30, seed=51)
    A = B + B.T + 4 * np.eye(30)
    y = dense_random(30, seed=52)[:, 2] * 3
    a = solve("bicor", DenseOp(A), y, 1e-12, 100, shadow=np.conj(y))
    b = solve("cocr", DenseOp(A), y, 1e-12, 100)
    assert a.iterations == b.iterations and a.status == CONVERGED
    np.testing.assert_allclose(a.history, b.history, rtol=1e-9, atol=1e-13 * a.history[0])


def test_cgne_error_monotone():
    A = dense_random(32, seed=61, shift=1.0)
    y = dense_random(32, seed=62)[:, 0]
    xs = np.linalg.solve(A, y)
    errs = []
    for k in range(1, 20):
        errs.append(np.linalg.norm(xs - solve("cgne", DenseOp(A), y, 0.0, k).x))
    assert all(b <= a * (1 + 1e-12) for a, b in zip(errs, errs[1:]))


# ---------------- direct solve, residuals, invariances ----------------
@pytest.mark.parametrize("n", [8, 16, 64])
@pytest.mark.parametrize("method", HOT_PATH)
def test_matches_lu(method, n):
    A = dense_random(n, seed=n + 5, shift=3 - 1j)
    rng = np.random.default_rng(n)
    xs = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = A @ xs
    res = solve(method, DenseOp(A), y, 1e-12, 10 * n)
    assert res.status == CONVERGED
    xl = lu_solve(A, y)
    assert np.linalg.norm(res.x - xl) <= 1e-9 * np.linalg.norm(xl)
    # true and recurrence residual agree
    assert res.true_rel_res <= 10 * 1e-12 and res.rec_rel_res <= 1e-12


@pytest.mark.parametrize("method", HOT_PATH)
def test_scale_invariance(method):
    A, y = cfg1(n=64, seed=3)
    c = 3 - 4j
    a = solve(method, DenseOp(A), y, 1e-10, 200)
    b = solve(method, DenseOp(c * A), c * y, 1e-10, 200)
    assert a.iterations == b.iterations
    assert np.linalg.norm(a.x - b.x) <= 1e-8 * np.linalg.norm(a.x)


def test_work_accounting():
    A, y = cfg1(n=64, seed=4)
    for m, (fa, fah) in {"bicgstab": (2, 0), "cgne": (1, 1), "qmr": (1, 1),
                          "bicor": (1, 1), "cors": (2, 0)}.items():
        res = solve(m, DenseOp(A), y, 0.0, 5)
        assert res.status == MAXIT and res.iterations == 5
        assert (res.matvecs_a, res.matvecs_ah) == (5 * fa, 5 * fah), m


def test_breakdown_fixture():
    A = np.array([[0, 1], [-1, 0]], dtype=np.complex128)
    y = np.array([1, 0], dtype=np.complex128)
    r = solve("bicgstab", DenseOp(A), y, 1e-10, 10)
    assert r.status == BREAKDOWN and r.breakdown == "sigma" and r.iterations == 0
    for m in ("bicor", "cors"):
        r = solve(m, DenseOp(A), y, 1e-10, 10)
        assert r.status == BREAKDOWN and r.breakdown == "rho", m


def test_zero_rhs_and_exact_x0_and_nonfinite():
    A, y = cfg1(n=16, seed=5)
    for m in HOT_PATH:
        r = solve(m, DenseOp(A), np.zeros(16, np.complex128), 1e-10, 10)
        assert r.status == CONVERGED and r.iterations == 0 and not np.any(r.x)
    xs = np.linalg.solve(A, y)
    r = solve("bicgstab", DenseOp(A), A @ xs, 1e-6, 10, x0=xs)
    assert r.status == CONVERGED and r.iterations <= 1
    yb = y.copy()
    yb[3] = np.nan
    r = solve("bicgstab", DenseOp(A), yb, 1e-10, 10)
    assert r.status == NONFINITE


@pytest.mark.parametrize("method", HOT_PATH)
def test_single_precision_stays_single(method):
    A, y = cfg1(n=64, seed=6)
    A, y = A.astype(np.complex64), y.astype(np.complex64)
    r = solve(method, DenseOp(A), y, 1e-5, 200)
    assert r.status == CONVERGED and r.x.dtype == np.complex64
    xs = np.linalg.solve(A.astype(np.complex128), y.astype(np.complex128))
    assert np.linalg.norm(r.x - xs) <= 1e-4 * np.linalg.norm(xs)
