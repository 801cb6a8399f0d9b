"""Pins for the SURVEY §8(f) NEXT-2 (iii) oracle: pipelined BiCGSTAB.  CPU only.

p-BiCGSTAB rewrites O1 with auxiliary recurrences (s = A p, z = A s, w = A r,
t = A w, v = A z) so that its two reduction phases do not precede the
products they feed.  In exact arithmetic it produces O1's iterates, so the
pin is equality with O1 in Gaussian-rational arithmetic at every k, plus
floating-point agreement, the half-step exit, special cases and breakdown.
"""

import numpy as np
import pytest

from oracle import solve, DenseOp
from oracle.solvers import CONVERGED, MAXIT, BREAKDOWN
from oracle.exact import to_exact
from oracle.direct import lu_solve
from workloads import dense_random, cfg1


def _rand_int(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.integers(-4, 5, (n, n)) + 1j * rng.integers(-4, 5, (n, n)) + 6 * np.eye(n)
    y = rng.integers(-3, 4, n) + 1j * rng.integers(-3, 4, n)
    return A.astype(np.complex128), y.astype(np.complex128)


@pytest.mark.parametrize("n", [3, 4, 5])
def test_pbicgstab_equals_bicgstab_exactly(n):
    A, y = _rand_int(n, seed=50 + n)
    Ae, ye = to_exact(A), to_exact(y)
    for k in range(1, n + 1):
        a = solve("pbicgstab", DenseOp(Ae), ye, 0.0, k)
        b = solve("bicgstab", DenseOp(Ae), ye, 0.0, k)
        assert a.status == b.status and a.iterations == b.iterations, k
        assert all(u == v for u, v in zip(a.x, b.x)), k
    a = solve("pbicgstab", DenseOp(Ae), ye, 0.0, n + 2)
    assert a.status == CONVERGED and a.half_step and a.iterations == n
    assert all(v == 0 for v in ye - DenseOp(Ae).apply(a.x))


def test_pbicgstab_floating_agreement_and_half_step():
    A, y = cfg1()
    a = solve("pbicgstab", DenseOp(A), y, 1e-10, 500)
    b = solve("bicgstab", DenseOp(A), y, 1e-10, 500)
    assert (a.status, a.iterations, a.half_step) == (b.status, b.iterations, b.half_step)
    assert np.linalg.norm(a.x - b.x) <= 1e-12 * np.linalg.norm(b.x)
    assert a.matvecs_a == 2 * a.iterations          # setup w, t; then v and, except at the exit, t
    B = dense_random(64, seed=9, shift=3 - 1j)
    yy = dense_random(64, seed=10)[:, 0]
    r = solve("pbicgstab", DenseOp(B), B @ yy, 1e-12, 200)
    assert r.status == CONVERGED and np.linalg.norm(r.x - lu_solve(B, B @ yy)) <= 1e-9 * np.linalg.norm(yy)


def test_pbicgstab_special_cases():
    c = 3 - 4j
    y = np.arange(10) + 1j * np.arange(10)[::-1]
    r = solve("pbicgstab", DenseOp(c * np.eye(10, dtype=np.complex128)), y, 1e-12, 50)
    assert r.status == CONVERGED and r.iterations == 1 and r.half_step
    np.testing.assert_allclose(r.x, y / c, rtol=1e-15)
    F = np.array([[0, 1], [-1, 0]], dtype=np.complex128)
    r = solve("pbicgstab", DenseOp(F), np.array([1, 0], np.complex128), 1e-10, 10)
    assert r.status == BREAKDOWN and r.breakdown == "sigma" and r.iterations == 0
    A, y = cfg1(n=64, seed=4)
    r = solve("pbicgstab", DenseOp(A), y, 0.0, 5)
    assert r.status == MAXIT and r.iterations == 5 and r.matvecs_a == 11
