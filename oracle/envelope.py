"""Rounding envelope of the oracle (SURVEY.md §8(c) "P-envelope").  TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

Krylov iterates are defined only in exact arithmetic; on rounding-sensitive
problems two correct implementations that differ only in summation order
legitimately disagree.  The envelope measures how far the
oracle itself moves under a rounding-sized perturbation: every matvec output
is multiplied elementwise by (1 + 2e-16·(ξ_re + iξ_im)), ξ iid N(0,1), for
seeds 1..E.  A GPU result is inside the envelope when its
iteration count lies in [k_min − 2, k_max + 2] and its x at equal iteration
count is within max(literal bar, 2·D) of the clean oracle, D being the largest
perturbed-vs-clean distance at that count.
"""

import numpy as np

from .solvers import solve


class NoisyOp:
    """Wraps an operator; perturbs every product output at relative size eps."""

    def __init__(self, op, seed, eps=None):
        self.op = op
        self.n = op.n
        self.dtype = op.dtype
        self.rng = np.random.default_rng(seed)
        self.eps = (2.0 * np.finfo(np.dtype(op.dtype)).eps if eps is None else eps)

    def _noise(self, v):
        xi = self.rng.standard_normal(len(v)) + 1j * self.rng.standard_normal(len(v))
        return (v * (1 + self.eps * xi)).astype(v.dtype)

    def apply(self, x):
        return self._noise(self.op.apply(x))

    def apply_h(self, x):
        return self._noise(self.op.apply_h(x))

    def apply_t(self, x):
        return self._noise(self.op.apply_t(x))

    def reset_counts(self):
        self.op.reset_counts()

    @property
    def n_a(self):
        return self.op.n_a

    @n_a.setter
    def n_a(self, v):
        self.op.n_a = v

    @property
    def n_ah(self):
        return self.op.n_ah


def iteration_envelope(method, op, y, tol, maxit, seeds=8):
    """(k_clean, k_min, k_max) over the clean run and `seeds` perturbed runs."""
    ks = [solve(method, op, y, tol, maxit).iterations]
    for s in range(1, seeds + 1):
        ks.append(solve(method, NoisyOp(op, s), y, tol, maxit).iterations)
    return ks[0], min(ks), max(ks)


def x_spread(method, op, y, k, seeds=8):
    """(x_clean(k), D(k)) — the clean iterate after exactly k iterations and the
    largest relative distance of a perturbed run's iterate from it."""
    xc = solve(method, op, y, 0.0, k).x
    nc = np.linalg.norm(xc)
    D = 0.0
    for s in range(1, seeds + 1):
        xs = solve(method, NoisyOp(op, s), y, 0.0, k).x
        D = max(D, float(np.linalg.norm(xs - xc) / nc))
    return xc, D
