"""Pins for the SURVEY §8(f) NEXT-3 oracle recurrences: BiCG, CGS, CGNR (P:57
§2.1) and COCR (§3.4).  CPU only.

Each is fixed by something other than itself:

* exact Gaussian-rational arithmetic: finite termination with A·x == y
  exactly at iteration n (generic A; complex-symmetric A for COCR);
* textbook reductions checked by dense linear algebra over an explicit Krylov
  basis: BiCG with shadow r₀ on Hermitian positive definite A is CG, whose
  iterate minimises the A-norm error over K_k(A, y); CGNR's iterate minimises
  ‖y − Ax‖ over K_k(AᴴA, Aᴴy); COCR on real symmetric A with a real right-hand
  side is CR, whose iterate minimises ‖y − Ax‖ over K_k(A, y);
* special cases (A = cI), the LU solution, scale invariance, work accounting,
  the breakdown fixture.

A dropped conjugation (e.g. conj(β) in BiCG's shadow update, or a conjugated
product in COCR) breaks the Krylov-minimisation or termination pins.
"""

import numpy as np
import pytest

from oracle import solve, DenseOp
from oracle.solvers import CONVERGED, MAXIT, BREAKDOWN, NEXT3
from oracle.exact import to_exact
from oracle.direct import lu_solve
from workloads import dense_random, cfg1


def _rand_int(n, seed, kind):
    rng = np.random.default_rng(seed)
    B = rng.integers(-4, 5, (n, n)) + 1j * rng.integers(-4, 5, (n, n))
    if kind == "hpd":
        A = B @ B.conj().T + np.eye(n)
    elif kind == "csym":
        A = B + B.T + 6 * np.eye(n)
    else:
        A = B + 6 * np.eye(n)
    y = rng.integers(-3, 4, n) + 1j * rng.integers(-3, 4, n)
    return A.astype(np.complex128), y.astype(np.complex128)


def _krylov(M, v, k):
    K = np.empty((len(v), k), dtype=np.complex128)
    K[:, 0] = v
    for j in range(1, k):
        K[:, j] = M @ K[:, j - 1]
    Q, _ = np.linalg.qr(K)
    return Q


@pytest.mark.parametrize("n", [3, 4, 5, 6])
@pytest.mark.parametrize("method,kind", [("bicg", "gen"), ("bicg", "hpd"), ("cgs", "gen"), ("cgs", "hpd"),
                                         ("cgnr", "gen"), ("cgnr", "hpd"), ("cocr", "csym")])
def test_exact_finite_termination(method, kind, n):
    A, y = _rand_int(n, seed=17 * n + len(kind), kind=kind)
    Ae, ye = to_exact(A), to_exact(y)
    op = DenseOp(Ae)
    res = solve(method, op, ye, 0.0, n + 3)
    assert res.status == CONVERGED, (res.status_name, res.breakdown)
    assert res.iterations <= n
    assert all(v == 0 for v in ye - op.apply(res.x)), "A·x must equal y exactly"
    if kind != "hpd":
        assert res.iterations == n


def test_bicg_is_cg_on_hpd():
    """BiCG, shadow r₀, Hermitian positive definite A = CG: x_k minimises
    (x − x*)ᴴA(x − x*) over K_k(A, y)  ⇔  (QᴴAQ)c = Qᴴy, x_k = Qc."""
    n = 40
    rng = np.random.default_rng(3)
    B = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    A = B @ B.conj().T / n + 0.5 * np.eye(n)
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for k in range(1, 9):
        res = solve("bicg", DenseOp(A), y, 0.0, k)
        assert res.iterations == k
        Q = _krylov(A, y, k)
        xm = Q @ np.linalg.solve(Q.conj().T @ A @ Q, Q.conj().T @ y)
        assert np.linalg.norm(res.x - xm) <= 1e-10 * np.linalg.norm(xm), k


def test_cgnr_minimises_residual_over_normal_krylov_space():
    n = 40
    A = dense_random(n, seed=71, shift=1.5 - 0.5j)
    y = dense_random(n, seed=72)[:, 0]
    prev = np.inf
    for k in range(1, 9):
        res = solve("cgnr", DenseOp(A), y, 0.0, k)
        assert res.iterations == k
        Q = _krylov(A.conj().T @ A, A.conj().T @ y, k)
        c, *_ = np.linalg.lstsq(A @ Q, y, rcond=None)
        xm = Q @ c
        assert np.linalg.norm(res.x - xm) <= 1e-9 * np.linalg.norm(xm), k
        rn = np.linalg.norm(y - A @ res.x)
        assert rn <= prev * (1 + 1e-12)
        prev = rn


@pytest.mark.parametrize("definite", [True, False])
def test_cocr_is_cr_on_real_symmetric(definite):
    """Real symmetric A (= Aᵀ = Aᴴ) and real y: [·,·] = ⟨·,·⟩ on the real
    iterates, COCR = CR = residual minimisation over K_k(A, y)."""
    n = 40
    rng = np.random.default_rng(11)
    B = rng.standard_normal((n, n))
    A = ((B + B.T) / 2 + (10 * np.eye(n) if definite else 0.2 * np.eye(n))).astype(np.complex128)
    y = rng.standard_normal(n).astype(np.complex128)
    for k in range(1, 9):
        res = solve("cocr", DenseOp(A), y, 0.0, k)
        assert res.iterations == k
        Q = _krylov(A, y, k)
        c, *_ = np.linalg.lstsq(A @ Q, y, rcond=None)
        xm = Q @ c
        assert np.linalg.norm(res.x - xm) <= 1e-9 * np.linalg.norm(xm), k


@pytest.mark.parametrize("method", NEXT3)
def test_scaled_identity_one_iteration(method):
    c = 3 - 4j
    n = 10
    rng = np.random.default_rng(0)
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    res = solve(method, DenseOp(c * np.eye(n, dtype=np.complex128)), y, 1e-12, 50)
    assert res.status == CONVERGED and res.iterations == 1
    np.testing.assert_allclose(res.x, y / c, rtol=1e-15, atol=1e-15)


@pytest.mark.parametrize("n", [8, 16, 64])
@pytest.mark.parametrize("method", NEXT3)
def test_matches_lu(method, n):
    A = dense_random(n, seed=n + 5, shift=3 - 1j)
    if method == "cocr":
        A = (A + A.T) / 2
    rng = np.random.default_rng(n)
    xs = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = A @ xs
    res = solve(method, DenseOp(A), y, 1e-12, 10 * n)
    assert res.status == CONVERGED
    xl = lu_solve(A, y)
    assert np.linalg.norm(res.x - xl) <= 1e-9 * np.linalg.norm(xl)
    assert res.true_rel_res <= 10 * 1e-12 and res.rec_rel_res <= 1e-12


@pytest.mark.parametrize("method", NEXT3)
def test_scale_invariance(method):
    A, y = cfg1(n=64, seed=3)
    if method == "cocr":
        A = (A + A.T) / 2
    c = 3 - 4j
    a = solve(method, DenseOp(A), y, 1e-10, 300)
    b = solve(method, DenseOp(c * A), c * y, 1e-10, 300)
    assert a.iterations == b.iterations
    assert np.linalg.norm(a.x - b.x) <= 1e-8 * np.linalg.norm(a.x)


def test_work_accounting():
    A, y = cfg1(n=64, seed=4)
    for m, want in {"bicg": (5, 5), "cgs": (10, 0), "cocr": (5, 0), "cgnr": (5, 5), "tfqmr": (10, 0),
                          "gmres": (5, 0), "bicgstabl": (9, 0)}.items():
        res = solve(m, DenseOp(A), y, 0.0, 5)
        assert res.status == MAXIT and res.iterations == 5
        assert (res.matvecs_a, res.matvecs_ah) == want, m


def test_breakdown_fixture():
    A = np.array([[0, 1], [-1, 0]], dtype=np.complex128)
    y = np.array([1, 0], dtype=np.complex128)
    for m, name in (("bicg", "sigma"), ("cgs", "sigma"), ("cocr", "rho"), ("tfqmr", "sigma"),
                    ("bicgstabl", "sigma")):
        r = solve(m, DenseOp(A), y, 1e-10, 10)
        assert r.status == BREAKDOWN and r.breakdown == name and r.iterations == 0, m
    r = solve("cgnr", DenseOp(A), y, 1e-10, 10)      # A unitary: CGNR converges at once
    assert r.status == CONVERGED and r.iterations == 1


# ---------------- TFQMR (§2.1) ----------------
def test_tfqmr_residual_bound_invariant():
    """Freund's bound ‖r_m‖ ≤ τ_m·√(m+1) (the quantity the stopping test uses)
    holds for the true residual after every pair and every half-step exit."""
    n = 60
    A = dense_random(n, seed=81, shift=1.5 + 0.5j)
    y = dense_random(n, seed=82)[:, 0]
    for k in range(1, 16):
        res = solve("tfqmr", DenseOp(A), y, 0.0, k)
        assert res.iterations == k
        bound = float(res.history[-1])
        true = np.linalg.norm(y - A @ res.x)
        assert true <= bound * (1 + 1e-9), (k, true, bound)
    # half-step exits too: a tolerance hit at the first half of a pair
    for tol in (1e-2, 1e-4, 1e-6, 1e-8):
        res = solve("tfqmr", DenseOp(A), y, tol, 200)
        assert res.status == CONVERGED
        assert np.linalg.norm(y - A @ res.x) <= float(res.history[-1]) * (1 + 1e-9)
        assert res.true_rel_res <= tol


@pytest.mark.parametrize("n", [4, 6])
def test_tfqmr_mpmath_termination(n):
    """100-digit arithmetic: the CGS polynomial it smooths terminates at
    iteration n, so does TFQMR (quasi-residual ~1e-95), with A·x = y."""
    mpmath = pytest.importorskip("mpmath")
    A, y = _rand_int(n, seed=300 + n, kind="gen")
    with mpmath.workdps(100):
        Am = np.array([[mpmath.mpc(complex(v)) for v in row] for row in A], dtype=object)
        ym = np.array([mpmath.mpc(complex(v)) for v in y], dtype=object)
        res = solve("tfqmr", DenseOp(Am), ym, 1e-90, n + 2)
        assert res.status == CONVERGED and res.iterations <= n
        r = ym - Am.dot(res.x)
        rel = mpmath.sqrt(sum(abs(v) ** 2 for v in r)) / mpmath.sqrt(sum(abs(v) ** 2 for v in ym))
        assert rel < mpmath.mpf("1e-85")


# ---------------- GMRES(m) (§2.1 "rgmres") ----------------
def _ls_krylov(A, r0, k):
    Q = _krylov(A, r0, k)
    c, *_ = np.linalg.lstsq(A @ Q, r0, rcond=None)
    return Q @ c


def test_gmres_is_krylov_least_squares_and_history_is_true_residual():
    """x_k = x₀ + argmin over K_k(A, r₀) of ‖y − A x‖ (dense least squares on a
    QR'd Krylov basis), and the Givens residual recorded in the history equals
    the true residual of x_k."""
    n = 50
    A = dense_random(n, seed=91, shift=1.0 + 1.0j)
    y = dense_random(n, seed=92)[:, 0]
    prev = np.inf
    for k in range(1, 12):
        res = solve("gmres", DenseOp(A), y, 0.0, k)
        assert res.iterations == k
        xm = _ls_krylov(A, y, k)
        assert np.linalg.norm(res.x - xm) <= 1e-9 * np.linalg.norm(xm), k
        true = np.linalg.norm(y - A @ res.x)
        assert abs(float(res.history[-1]) - true) <= 1e-10 * np.linalg.norm(y), k
        assert true <= prev * (1 + 1e-12)
        prev = true


def test_gmres_restart_restarts_from_the_current_iterate():
    """GMRES(4): after a restart at x₄ the next iterates are x₄ + argmin over
    K_j(A, y − A x₄); the restart costs one extra product."""
    n = 40
    A = dense_random(n, seed=93, shift=2.0 - 0.5j)
    y = dense_random(n, seed=94)[:, 0]
    x4 = solve("gmres", DenseOp(A), y, 0.0, 4, restart=4).x
    r4 = y - A @ x4
    for j in range(1, 4):
        res = solve("gmres", DenseOp(A), y, 0.0, 4 + j, restart=4)
        assert res.iterations == 4 + j and res.matvecs_a == 4 + j + 1
        xm = x4 + _ls_krylov(A, r4, j)
        assert np.linalg.norm(res.x - xm) <= 1e-9 * np.linalg.norm(xm), j


@pytest.mark.parametrize("n", [4, 6])
def test_gmres_mpmath_termination(n):
    mpmath = pytest.importorskip("mpmath")
    A, y = _rand_int(n, seed=400 + n, kind="gen")
    with mpmath.workdps(100):
        Am = np.array([[mpmath.mpc(complex(v)) for v in row] for row in A], dtype=object)
        ym = np.array([mpmath.mpc(complex(v)) for v in y], dtype=object)
        res = solve("gmres", DenseOp(Am), ym, 1e-90, n + 2)
        assert res.status == CONVERGED and res.iterations == n
        r = ym - Am.dot(res.x)
        rel = mpmath.sqrt(sum(abs(v) ** 2 for v in r)) / mpmath.sqrt(sum(abs(v) ** 2 for v in ym))
        assert rel < mpmath.mpf("1e-85")


def test_gmres_cgs2_keeps_the_givens_residual_true():
    """Ill-conditioned A (eigenvalues over 8 decades): with the second
    Gram–Schmidt pass (R13) the Givens residual stays the true residual to
    ~2e-13 over 60 steps; one pass drifts to ~1.4e-12 (loss of orthogonality)."""
    n = 120
    rng = np.random.default_rng(5)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    A = (Q * (np.logspace(0, 8, n) * np.exp(1j * rng.uniform(0, 0.3, n)))) @ Q.conj().T
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    res = solve("gmres", DenseOp(A), y, 0.0, 60, restart=60)
    gap = abs(float(res.history[-1]) - np.linalg.norm(y - A @ res.x)) / np.linalg.norm(y)
    assert gap <= 6e-13


# ---------------- BiCGstab(ℓ) (§3.1) ----------------
def test_bicgstabl_one_is_bicgstab():
    """ℓ = 1: the minimal-residual part is BiCGSTAB's ω step — same iterates
    and the same number of products at every k."""
    A = dense_random(40, seed=101, shift=1.5 - 1j)
    y = dense_random(40, seed=102)[:, 0]
    for k in range(1, 11):
        a = solve("bicgstabl", DenseOp(A), y, 0.0, k, ell=1)
        b = solve("bicgstab", DenseOp(A), y, 0.0, k)
        assert a.matvecs_a == b.matvecs_a == 2 * k
        assert np.linalg.norm(a.x - b.x) <= 1e-13 * np.linalg.norm(b.x), k
    a = solve("bicgstabl", DenseOp(A), y, 1e-10, 200, ell=1)
    b = solve("bicgstab", DenseOp(A), y, 1e-10, 200)
    assert (a.iterations, a.matvecs_a) == (b.iterations, b.matvecs_a)     # incl. the half-step exit


@pytest.mark.parametrize("n", [3, 4, 5, 6])
@pytest.mark.parametrize("ell", [1, 2, 3])
def test_bicgstabl_exact_finite_termination(ell, n):
    A, y = _rand_int(n, seed=23 * n + ell, kind="gen")
    Ae, ye = to_exact(A), to_exact(y)
    op = DenseOp(Ae)
    res = solve("bicgstabl", op, ye, 0.0, n + 3 * ell, ell=ell)
    assert res.status == CONVERGED, (res.status_name, res.breakdown)
    assert res.iterations <= n
    assert all(v == 0 for v in ye - op.apply(res.x)), "A·x must equal y exactly"


def test_bicgstabl_mr_part_minimises_over_the_cycle_space():
    """After every cycle the MR update leaves r̂₀ orthogonal to r̂₁..r̂_ℓ (the
    normal equations of the minimal-residual polynomial), the invariants
    r̂_j = A r̂_{j−1}, û_j = A û_{j−1} hold, and r̂₀ is the residual y − A x."""
    A = dense_random(50, seed=105, shift=2 + 1j)
    y = dense_random(50, seed=106)[:, 0]
    for ell in (2, 3, 4):
        cycles = []
        res = solve("bicgstabl", DenseOp(A), y, 0.0, 4 * ell, ell=ell,
                    trace=lambda R, U: cycles.append(([v.copy() for v in R], [v.copy() for v in U])))
        assert len(cycles) == 4
        for R, U in cycles:
            nr = np.linalg.norm(R[0])
            for j in range(1, ell + 1):
                assert abs(np.vdot(R[j], R[0])) <= 1e-10 * np.linalg.norm(R[j]) * nr, (ell, j)
                if j < ell:
                    assert np.linalg.norm(R[j + 1] - A @ R[j]) <= 1e-10 * np.linalg.norm(R[j + 1])
                    assert np.linalg.norm(U[j + 1] - A @ U[j]) <= 1e-10 * np.linalg.norm(U[j + 1])
        assert np.linalg.norm(cycles[-1][0][0] - (y - A @ res.x)) <= 1e-10 * np.linalg.norm(y)


# ---------------- right Jacobi preconditioning (NEXT-4) ----------------
def test_jacobi_constant_diagonal_is_a_rescaling():
    """d = c·1: B = A/c, u = c·x — the same iterates (scale invariance)."""
    from oracle import solve_jacobi
    A, y = cfg1(n=64, seed=8)
    for m in ("bicgstab", "qmr", "gmres"):
        a = solve(m, DenseOp(A), y, 1e-10, 300)
        b = solve_jacobi(m, DenseOp(A), np.full(64, 3 - 4j), y, 1e-10, 300)
        assert a.iterations == b.iterations
        assert np.linalg.norm(a.x - b.x) <= 1e-9 * np.linalg.norm(a.x), m


def test_jacobi_diagonal_matrix_one_iteration_and_badly_scaled_speedup():
    from oracle import solve_jacobi
    rng = np.random.default_rng(12)
    n = 80
    d = np.logspace(0, 4, n) * np.exp(1j * rng.uniform(0, 2 * np.pi, n))
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    r = solve_jacobi("bicgstab", DenseOp(np.diag(d)), d, y, 1e-12, 10)
    assert r.status == CONVERGED and r.iterations == 1
    np.testing.assert_allclose(r.x, y / d, rtol=1e-13)
    A = np.diag(d) + 0.3 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    plain = solve("bicgstab", DenseOp(A), y, 1e-10, 2000)
    pre = solve_jacobi("bicgstab", DenseOp(A), d, y, 1e-10, 2000)
    assert pre.status == CONVERGED and pre.iterations <= 20               # unpreconditioned: > 2000 (MAXIT)
    assert plain.status != CONVERGED or plain.iterations >= 10 * pre.iterations
    xl = lu_solve(A, y)
    assert np.linalg.norm(pre.x - xl) <= 1e-8 * np.linalg.norm(xl)
    assert np.linalg.norm(y - A @ pre.x) / np.linalg.norm(y) <= 1e-9
