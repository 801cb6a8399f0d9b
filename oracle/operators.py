"""The user operator: ``matvec`` / ``cmatvec``.  TEST INFRASTRUCTURE ONLY.

P:95 (§5): "All the communication to matvec, cmatvec is set in module
arraymodule.  User can implement his/her own sparse matrix scheme in matvec
and cmatvec."  P:17 (abstract): the matrix-vector product is "separated from
the conjugate gradient iterations itself".

Each operator exposes

* ``apply(x)``   = A·x                 (matvec)
* ``apply_h(x)`` = Aᴴ·x                (cmatvec)
* ``apply_t(x)`` = Aᵀ·x (unconjugated)

and counts its applications (work accounting).

Dense storage is row-major.  Aᴴx is formed as conj(conj(x)ᵀ·A) so that the
matrix is never copied or conjugated.  CSR uses
scipy.sparse for floating dtypes (library primitive) and a plain double loop
for object dtypes (exact / mpmath modes) and the CSR pins.
"""

import numpy as np


class _Counted:
    def __init__(self):
        self.n_a = 0
        self.n_ah = 0
        self.n_at = 0

    def reset_counts(self):
        self.n_a = self.n_ah = self.n_at = 0


class DenseOp(_Counted):
    """Dense row-major n×n operator."""

    def __init__(self, A):
        super().__init__()
        A = np.asarray(A)
        if A.ndim != 2 or A.shape[0] != A.shape[1]:
            raise ValueError("DenseOp needs a square matrix")
        self.A = A
        self.n = A.shape[0]
        self.dtype = A.dtype

    def apply(self, x):
        self.n_a += 1
        return self.A.dot(x)

    def apply_h(self, x):
        self.n_ah += 1
        return np.conj(np.conj(x).dot(self.A))

    def apply_t(self, x):
        self.n_at += 1
        return x.dot(self.A)


class CsrOp(_Counted):
    """CSR operator: rowptr (n+1), colind (nnz), vals (nnz)."""

    def __init__(self, rowptr, colind, vals, n=None):
        super().__init__()
        self.rowptr = np.asarray(rowptr)
        self.colind = np.asarray(colind)
        self.vals = np.asarray(vals)
        self.n = len(self.rowptr) - 1 if n is None else n
        self.dtype = self.vals.dtype
        if self.vals.dtype != object:
            import scipy.sparse as sp
            self._M = sp.csr_matrix((self.vals, self.colind, self.rowptr),
                                    shape=(self.n, self.n))
        else:
            self._M = None

    def _loop(self, x, conj_vals, transpose):
        out = np.zeros(self.n, dtype=x.dtype) if x.dtype != object else \
            np.array([0] * self.n, dtype=object)
        for i in range(self.n):
            for k in range(self.rowptr[i], self.rowptr[i + 1]):
                v = self.vals[k]
                if conj_vals:
                    v = v.conjugate()
                j = self.colind[k]
                if transpose:
                    out[j] = out[j] + v * x[i]
                else:
                    out[i] = out[i] + v * x[j]
        return out

    def apply(self, x):
        self.n_a += 1
        if self._M is None:
            return self._loop(x, False, False)
        return self._M.dot(x)

    def apply_h(self, x):
        self.n_ah += 1
        if self._M is None:
            return self._loop(x, True, True)
        return np.conj(self._M.T.dot(np.conj(x)))

    def apply_t(self, x):
        self.n_at += 1
        if self._M is None:
            return self._loop(x, False, True)
        return self._M.T.dot(x)

    def apply_loop(self, x, op="A"):
        """Plain double-loop product (no scipy) — used to pin the scipy path."""
        return self._loop(x, op == "AH", op in ("AH", "AT"))

    def to_dense(self):
        D = np.zeros((self.n, self.n), dtype=self.vals.dtype)
        for i in range(self.n):
            for k in range(self.rowptr[i], self.rowptr[i + 1]):
                D[i, self.colind[k]] += self.vals[k]
        return D


class ToeplitzOp(_Counted):
    """3-level Toeplitz operator on an nx × ny × nz lattice (x fastest, unit
    spacing): (A x)_i = d·x_i + Σ_{j≠i} K(r_i − r_j)·x_j — the discrete-dipole
    structure of P:47 (§1) (BJ:8, BJ:10 configs are scalar instances).

    The lattice sum is a linear convolution; this oracle evaluates it with a
    library FFT (scipy.fft, a step of the definition) on the zero-padded
    (2nz, 2ny, 2nx) box, in the working precision of ``kernel``.
    ``kernel[dz+nz-1, dy+ny-1, dx+nx-1]`` = K(dx, dy, dz); the δ = 0 entry is
    ignored.  Aᵀ convolves with K(−δ); Aᴴx = conj(Aᵀ conj(x)).  Pinned against
    the dense definition (tests/test_oracle_numerics.py)."""

    def __init__(self, kernel, dims, diag):
        import scipy.fft as sf
        super().__init__()
        self._fft = sf
        nx, ny, nz = dims
        K = np.array(kernel).reshape(2 * nz - 1, 2 * ny - 1, 2 * nx - 1).copy()
        K[nz - 1, ny - 1, nx - 1] = 0
        self.dims = dims
        self.n = nx * ny * nz
        self.dtype = K.dtype
        self.diag = self.dtype.type(diag)
        self.Kh = self._embed_fft(K)
        self.Kh_t = self._embed_fft(K[::-1, ::-1, ::-1])      # K(−δ)

    def _embed_fft(self, K):
        nx, ny, nz = self.dims
        C = np.zeros((2 * nz, 2 * ny, 2 * nx), dtype=self.dtype)
        # circulant index m ↔ displacement m (m < n) or m − 2n (m > n); m = n unused
        idx = [np.r_[0:n, n + 1:2 * n] for n in (nz, ny, nx)]
        src = [np.r_[n - 1:2 * n - 1, 0:n - 1] for n in (nz, ny, nx)]
        C[np.ix_(*idx)] = K[np.ix_(*src)]
        return self._fft.fftn(C)

    def _conv(self, x, Kh):
        nx, ny, nz = self.dims
        X = np.zeros((2 * nz, 2 * ny, 2 * nx), dtype=self.dtype)
        X[:nz, :ny, :nx] = np.asarray(x).reshape(nz, ny, nx)
        return self._fft.ifftn(self._fft.fftn(X) * Kh)[:nz, :ny, :nx].ravel().astype(self.dtype)

    def apply(self, x):
        self.n_a += 1
        return self.diag * x + self._conv(x, self.Kh)

    def apply_t(self, x):
        self.n_at += 1
        return self.diag * x + self._conv(x, self.Kh_t)

    def apply_h(self, x):
        self.n_ah += 1
        xc = np.conj(x)
        return np.conj(self.diag * xc + self._conv(xc, self.Kh_t))


class JacobiRightOp(_Counted):
    """Right Jacobi preconditioning: the operator
    B = A·D⁻¹ with D = diag(d) — B·v = A(D⁻¹v), Bᴴ·v = D⁻ᴴ(Aᴴv), Bᵀ·v = D⁻¹(Aᵀv).
    A solve of B u = y gives x = D⁻¹u; the residual y − B u = y − A x is the
    original system's, so the common stopping rule is unchanged."""

    def __init__(self, op, d):
        super().__init__()
        self.op = op
        self.dinv = 1.0 / np.asarray(d)
        self.n = op.n

    def apply(self, x):
        self.n_a += 1
        return self.op.apply(self.dinv * x)

    def apply_h(self, x):
        self.n_ah += 1
        return np.conj(self.dinv) * self.op.apply_h(x)

    def apply_t(self, x):
        self.n_at += 1
        return self.dinv * self.op.apply_t(x)


def reference_apply(A, x, op="A"):
    """Per-matvec parity reference.

    Accumulated more accurately than the working precision: complex64
    inputs are promoted to complex128 and the product is taken with numpy
    (BLAS zgemv); complex128 inputs go straight to zgemv.  ``A`` may be a
    dense array or a CsrOp."""
    if isinstance(A, CsrOp):
        op_ = CsrOp(A.rowptr, A.colind, A.vals.astype(np.complex128), A.n)
        xx = np.asarray(x, dtype=np.complex128)
        return {"A": op_.apply, "AH": op_.apply_h, "AT": op_.apply_t}[op](xx)
    A = np.asarray(A)
    xx = np.asarray(x, dtype=np.complex128)
    AA = A.astype(np.complex128, copy=False)
    if op == "A":
        return AA.dot(xx)
    if op == "AH":
        return np.conj(np.conj(xx).dot(AA))
    if op == "AT":
        return xx.dot(AA)
    raise ValueError(op)


def check_complex_symmetric(A, tol=0.0):
    """max|A_ij − A_ji| ≤ tol·max|A| (unconjugated)."""
    A = np.asarray(A)
    m = np.max(np.abs(A)) if A.size else 0.0
    return bool(np.max(np.abs(A - A.T)) <= tol * m) if A.size else True
