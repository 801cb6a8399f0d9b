"""Complex vector primitives.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:47 (§1): "I have removed calls to BLAS ... in favor of FORTRAN90 intrinsics
such as dot_product or sum".  For complex arguments F90 ``dot_product(u, v)``
conjugates its first argument, ``sum(u*v)`` does not:

* dotc(u, v) = Σ conj(u_i)·v_i
* dotu(u, v) = Σ u_i·v_i
* norm2(u)   = sqrt(Re dotc(u, u))
* norm_sq(u) = Re dotc(u, u)

Floating arrays use numpy's ``vdot`` / ``dot`` (a library primitive for the
plain sum); object arrays (exact / mpmath modes) use a plain Python loop.
"""

import math
from fractions import Fraction

import numpy as np


def _is_obj(u):
    return getattr(u, "dtype", None) == object


def _check(u, v):
    if len(u) != len(v):
        raise ValueError(f"dimension mismatch: {len(u)} vs {len(v)}")


def dotc(u, v):
    """Σ conj(u_i)·v_i  (F90 dot_product on complex)."""
    _check(u, v)
    if _is_obj(u) or _is_obj(v):
        acc = 0
        for a, b in zip(u, v):
            acc = acc + a.conjugate() * b
        return acc
    return np.vdot(u, v)


def dotu(u, v):
    """Σ u_i·v_i, no conjugation  (F90 sum(u*v))."""
    _check(u, v)
    if _is_obj(u) or _is_obj(v):
        acc = 0
        for a, b in zip(u, v):
            acc = acc + a * b
        return acc
    return np.dot(u, v)


def norm_sq(u):
    """Re Σ |u_i|²  (the real part of dotc(u, u))."""
    s = dotc(u, u)
    return s.real


def sqrt(x):
    """Square root in the scalar's own precision (float32/float64/mpf)."""
    try:
        import mpmath
        if isinstance(x, (mpmath.mpf, mpmath.mpc)):
            return mpmath.sqrt(x)
    except ImportError:  # pragma: no cover
        pass
    if isinstance(x, Fraction):          # exact mode: histories are diagnostics
        return math.sqrt(x)
    return np.sqrt(x)


def norm2(u):
    """sqrt(Re dotc(u, u))."""
    return sqrt(norm_sq(u))
