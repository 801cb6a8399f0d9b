"""Independent dense direct solver.  TEST INFRASTRUCTURE ONLY.

S:466-508 (module "oracle"): dense LU with partial pivoting and the relative
residual.  Plain Doolittle elimination with row interchanges, written out —
no shared code with the iterative solvers.  Used at n ≤ 64 (the
north_star's "dense Gaussian-elimination solves on n≤64") and cross-checked
against LAPACK (numpy.linalg.solve) in the tests.
"""

import numpy as np


class SingularMatrix(ArithmeticError):
    pass


def lu_factor(A):
    """PA = LU, partial pivoting.  Returns (LU, perm)."""
    LU = np.array(A, dtype=np.complex128, copy=True)
    n = LU.shape[0]
    perm = np.arange(n)
    scale = np.max(np.abs(LU)) if n else 0.0
    for k in range(n):
        p = k + int(np.argmax(np.abs(LU[k:, k])))
        if abs(LU[p, k]) <= np.finfo(np.float64).eps * n * scale:
            raise SingularMatrix(f"pivot {k} is (numerically) zero")
        if p != k:
            LU[[k, p], :] = LU[[p, k], :]
            perm[[k, p]] = perm[[p, k]]
        for i in range(k + 1, n):
            LU[i, k] = LU[i, k] / LU[k, k]
            for j in range(k + 1, n):
                LU[i, j] = LU[i, j] - LU[i, k] * LU[k, j]
    return LU, perm


def lu_solve(A, y):
    """x with Ax = y by forward/back substitution on the LU factors."""
    LU, perm = lu_factor(A)
    n = LU.shape[0]
    b = np.asarray(y, dtype=np.complex128)[perm]
    z = np.zeros(n, dtype=np.complex128)
    for i in range(n):
        s = b[i]
        for j in range(i):
            s = s - LU[i, j] * z[j]
        z[i] = s
    x = np.zeros(n, dtype=np.complex128)
    for i in range(n - 1, -1, -1):
        s = z[i]
        for j in range(i + 1, n):
            s = s - LU[i, j] * x[j]
        x[i] = s / LU[i, i]
    return x


def rel_residual(apply, x, y, denom=None):
    """‖y − A·x‖₂ / denom, denom = ‖y‖₂ by default."""
    r = np.asarray(y) - apply(x)
    d = np.linalg.norm(y) if denom is None else denom
    if d == 0:
        raise ZeroDivisionError("zero denominator")
    return float(np.linalg.norm(r) / d)
