"""CPU oracle for the CCGPAK complex-Krylov hot path (arXiv:1208.4869).

TEST INFRASTRUCTURE ONLY.  Nothing under ``oracle/`` is part of the product.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
leg / ``--impl reference`` arm may import it.  The product path
(``paper_1208_4869_b200``) never imports it and shares no code with it: no
kernels, no helpers, no constants.  The only module both sides consume is
``workloads/`` (seeded input generators, which hold none of the method's
arithmetic).

What it computes (PAPER.md = "P:<line>", SPEC.md = "S:<line>"):

* ``numerics``  - dotc / dotu / norm2, the F90 ``dot_product`` / ``sum(u*v)``
  intrinsics the paper substitutes for BLAS (§1).
* ``operators`` - the user ``matvec`` / ``cmatvec`` of ``arraymodule`` (§5):
  A·x, Aᴴ·x, Aᵀ·x for dense and CSR storage, and the lattice
  (3-level Toeplitz, DDA-structured) operator via a library FFT.
* ``solvers``   - BiCGSTAB, CGNE, QMR (PIM90 set, §2.1; §6) and
  BiCOR / CORS (§2.4), written step by step in the notation of
  SURVEY.md §8(c) O1-O5, plus BiCG, CGS, CGNR and COCR (§3.4),
  the SURVEY §8(f) NEXT-3 rows (also equivalence pins for BiCOR / CORS).
* ``direct``    - dense LU with partial pivoting and the relative residual
  (S:466-508), the independent direct-solve check.

The scalar type is generic: numpy complex64/complex128 arrays run in the
working precision ("simple to switch between single and double
precisions"), numpy ``object`` arrays of ``exact.GaussianRational``
run in exact arithmetic, and object arrays of ``mpmath.mpc`` run in
arbitrary precision.  These two extra modes exist only to pin the oracle
(finite termination, SURVEY.md §8(c) pin table).

Parity pins: every function here is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py``.  No function is
"parity unpinned".
"""

from . import numerics, operators, solvers, direct, exact  # noqa: F401
from .solvers import solve, solve_jacobi, Result, METHODS  # noqa: F401
from .operators import DenseOp, CsrOp, ToeplitzOp, JacobiRightOp  # noqa: F401
