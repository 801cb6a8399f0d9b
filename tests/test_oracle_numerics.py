"""Pins for oracle.numerics / oracle.operators / oracle.direct (CPU only).

Each check is against something other than the oracle itself: the worked
examples SPEC.md prints (tests/golden/spec_examples.json, cited per entry),
exact rational arithmetic, exactly-rounded sums (math.fsum), closed-form
eigenvectors, LAPACK, and algebraic identities.
"""

import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import numerics as nm
from oracle.operators import DenseOp, CsrOp, reference_apply, check_complex_symmetric
from oracle.direct import lu_solve, rel_residual, SingularMatrix
from oracle.exact import GaussianRational as GR, to_exact
from workloads import helmholtz_csr, dense_random


def C(v):
    return np.array([complex(a, b) for a, b in v], dtype=np.complex128)


def CM(m):
    return np.array([[complex(a, b) for a, b in row] for row in m], dtype=np.complex128)


# ---------------- worked examples ----------------
def test_dotc_examples(golden):
    for e in golden["dotc"]:
        assert nm.dotc(C(e["u"]), C(e["v"])) == complex(*e["out"]), e["cite"]


def test_dotu_examples(golden):
    for e in golden["dotu"]:
        assert nm.dotu(C(e["u"]), C(e["v"])) == complex(*e["out"]), e["cite"]


def test_norm2_examples(golden):
    for e in golden["norm2"]:
        assert nm.norm2(C(e["u"])) == e["out"], e["cite"]


def test_apply_examples(golden):
    for e in golden["apply"]:
        x = C(e["x"])
        if "csr" in e:
            c = e["csr"]
            op = CsrOp(c["rowptr"], c["colind"], C(c["vals"]))
        else:
            op = DenseOp(CM(e["A"]))
        f = {"A": op.apply, "AH": op.apply_h, "AT": op.apply_t}[e["op"]]
        np.testing.assert_array_equal(f(x), C(e["out"]), err_msg=e["cite"])


def test_complex_symmetric_examples(golden):
    for e in golden["complex_symmetric"]:
        assert check_complex_symmetric(CM(e["A"]), e["tol"]) == e["out"], e["cite"]
    B = dense_random(9, seed=3)
    assert check_complex_symmetric(B + B.T, 1e-14)


def test_lu_examples(golden):
    for e in golden["lu_solve"]:
        np.testing.assert_allclose(lu_solve(CM(e["A"]), C(e["y"])), C(e["out"]),
                                   rtol=0, atol=1e-15, err_msg=e["cite"])
    for e in golden["rel_residual"]:
        op = DenseOp(CM(e["A"]))
        assert rel_residual(op.apply, C(e["x"]), C(e["y"])) == pytest.approx(e["out"]), e["cite"]


# ---------------- invariants ----------------
def test_dot_symmetries():
    rng = np.random.default_rng(5)
    u = rng.standard_normal(37) + 1j * rng.standard_normal(37)
    v = rng.standard_normal(37) + 1j * rng.standard_normal(37)
    assert nm.dotc(u, v) == pytest.approx(np.conj(nm.dotc(v, u)), rel=1e-15)
    assert nm.dotu(u, v) == pytest.approx(nm.dotu(v, u), rel=1e-15)
    assert nm.dotc(u, u).imag == 0 and nm.dotc(u, u).real > 0


def test_dots_exact_rational():
    """The float path equals the exact rational sum on small-integer data."""
    rng = np.random.default_rng(1)
    u = (rng.integers(-9, 10, 50) + 1j * rng.integers(-9, 10, 50)).astype(np.complex128)
    v = (rng.integers(-9, 10, 50) + 1j * rng.integers(-9, 10, 50)).astype(np.complex128)
    ue, ve = to_exact(u), to_exact(v)
    ex = nm.dotc(ue, ve)
    assert complex(ex) == nm.dotc(u, v)
    ex = nm.dotu(ue, ve)
    assert complex(ex) == nm.dotu(u, v)
    # hand expansion of the definition for one pair of exact scalars
    assert GR(1, 2).conjugate() * GR(2, 0) + GR(3, 0).conjugate() * GR(0, 1) == GR(2, -1)


def test_dtype_is_working_precision():
    u = np.ones(8, np.complex64)
    assert nm.dotc(u, u).dtype == np.complex64
    assert nm.norm2(u).dtype == np.float32


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_adjoint_identities(dtype):
    n = 61
    A = dense_random(n, seed=2, dtype=dtype, shift=1.0)
    rng = np.random.default_rng(3)
    x = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(dtype)
    z = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(dtype)
    op = DenseOp(A)
    eps = np.finfo(dtype).eps
    slack = 8 * eps * n * np.max(np.abs(A)) * np.linalg.norm(x) * np.linalg.norm(z)
    assert abs(nm.dotc(z, op.apply(x)) - nm.dotc(op.apply_h(z), x)) <= slack
    assert abs(nm.dotu(z, op.apply(x)) - nm.dotu(op.apply_t(z), x)) <= slack
    # Aᵀx = conj(Aᴴ conj x)
    np.testing.assert_allclose(op.apply_t(x), np.conj(op.apply_h(np.conj(x))),
                               rtol=0, atol=10 * eps * n)


def test_dense_matches_exactly_rounded_rows():
    """reference_apply rows vs math.fsum of the exact products (brute force)."""
    n = 300
    A = dense_random(n, seed=11, dtype=np.complex64, shift=2 + 0.3j)
    rng = np.random.default_rng(12)
    x = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
    for op in ("A", "AH", "AT"):
        y = reference_apply(A, x, op)
        M = A.astype(np.complex128)
        if op == "AH":
            M = M.conj().T
        elif op == "AT":
            M = M.T
        for i in (0, 1, 149, n - 1):
            re = math.fsum([(M[i, j] * x[j]).real for j in range(n)])
            im = math.fsum([(M[i, j] * x[j]).imag for j in range(n)])
            # c64 inputs: each product is exact in fp64 -> only the BLAS sum rounds
            assert abs(y[i] - complex(re, im)) <= 1e-13 * np.sum(np.abs(M[i]) * np.abs(x))


def test_csr_scipy_equals_plain_loop_and_dense():
    rp, ci, v = helmholtz_csr(N=6, kh=10 / 6)
    op = CsrOp(rp, ci, v)
    D = op.to_dense()
    rng = np.random.default_rng(4)
    x = rng.standard_normal(op.n) + 1j * rng.standard_normal(op.n)
    for o, f in (("A", op.apply), ("AH", op.apply_h), ("AT", op.apply_t)):
        ref = {"A": D, "AH": D.conj().T, "AT": D.T}[o] @ x
        np.testing.assert_allclose(f(x), ref, rtol=1e-14, atol=1e-13)
        np.testing.assert_allclose(op.apply_loop(x, o), ref, rtol=1e-14, atol=1e-13)


def test_helmholtz_closed_form_eigenvectors():
    """v = ⊗ sin(π m_d i_d/(N+1)) satisfies Av = λv, λ = Σ 2(1−cos(π m_d/(N+1))) − k²(1+i/2)."""
    N, kh = 12, 10.0 / 12
    rp, ci, v = helmholtz_csr(N=N, kh=kh)
    op = CsrOp(rp, ci, v)
    idx = np.arange(1, N + 1)
    for m in ((1, 1, 1), (2, 5, 7), (12, 1, 3)):
        s = [np.sin(np.pi * md * idx / (N + 1)) for md in m]
        vec = np.einsum("k,j,i->kji", s[2], s[1], s[0]).reshape(-1).astype(np.complex128)
        lam = sum(2 * (1 - np.cos(np.pi * md / (N + 1))) for md in m) - kh * kh * (1 + 0.5j)
        res = op.apply(vec) - lam * vec
        assert np.linalg.norm(res) <= 1e-13 * np.linalg.norm(vec) * 12
    # exact constants (Q11): diagonal 6 - k²(1 + i/2) with k = 10/128
    _, _, v128 = helmholtz_csr(N=4, kh=10 / 128)
    assert complex(6 - 25 / 4096, -25 / 8192) in set(v128.tolist())


def test_lu_vs_lapack_and_singular():
    for n in (1, 7, 33, 64):
        A = dense_random(n, seed=n, shift=1.5)
        y = np.arange(n) + 1j
        np.testing.assert_allclose(lu_solve(A, y), np.linalg.solve(A, y), rtol=1e-11, atol=1e-12)
    with pytest.raises(SingularMatrix):
        lu_solve(np.array([[1, 2], [2, 4]], dtype=np.complex128), np.ones(2))


def test_exact_scalar():
    a, b = GR(1, 2), GR(3, -4)
    assert a / b * b == a
    assert (a * b).conjugate() == a.conjugate() * b.conjugate()
    assert GR(Fraction(1, 3), 0) * 3 == 1


# ---------------- the lattice (3-level Toeplitz) operator ----------------
def _dense_from_kernel(K, dims, diag):
    """Brute force: A[i, j] = K(r_i − r_j), A[i, i] = diag, by explicit loops."""
    nx, ny, nz = dims
    n = nx * ny * nz
    A = np.empty((n, n), dtype=np.complex128)
    for i in range(n):
        xi, yi, zi = i % nx, (i // nx) % ny, i // (nx * ny)
        for j in range(n):
            xj, yj, zj = j % nx, (j // nx) % ny, j // (nx * ny)
            A[i, j] = diag if i == j else K[zi - zj + nz - 1, yi - yj + ny - 1, xi - xj + nx - 1]
    return A


def test_toeplitz_op_matches_dense_definition():
    """Random non-symmetric kernel on a non-cubic lattice: A·x, Aᴴ·x, Aᵀ·x of
    the FFT operator equal the brute-force dense matrix's products."""
    from oracle import ToeplitzOp, DenseOp
    dims = (5, 3, 4)
    rng = np.random.default_rng(5)
    K = rng.standard_normal((7, 5, 9)) + 1j * rng.standard_normal((7, 5, 9))
    op = ToeplitzOp(K, dims, 2 - 1j)
    A = _dense_from_kernel(K, dims, 2 - 1j)
    x = rng.standard_normal(60) + 1j * rng.standard_normal(60)
    for f, ref in ((op.apply, A @ x), (op.apply_t, A.T @ x), (op.apply_h, A.conj().T @ x)):
        assert np.linalg.norm(f(x) - ref) <= 1e-14 * np.linalg.norm(ref)


def test_dda_kernel_matches_lattice_rows_and_cfg2():
    """dda_kernel holds exactly the off-diagonal entries of dda_lattice_rows;
    the FFT operator reproduces config 2's dense product."""
    from oracle import ToeplitzOp, DenseOp
    from workloads import dda_kernel, dda_lattice_rows, cfg2
    dims = (4, 3, 5)
    K = dda_kernel(dims, 0.7)
    A = dda_lattice_rows(dims, 0.7, 2.5 + 0.2j, 0, 60)
    assert np.array_equal(_dense_from_kernel(K, dims, 2.5 + 0.2j), A)
    A2, y2 = cfg2()
    op = ToeplitzOp(dda_kernel((16, 16, 16), 1.0), (16, 16, 16), 3 + 0.5j)
    assert np.linalg.norm(op.apply(y2) - A2 @ y2) <= 2e-15 * np.linalg.norm(A2 @ y2)
    assert np.linalg.norm(op.apply_h(y2) - A2.conj().T @ y2) <= 2e-15 * np.linalg.norm(A2 @ y2)
