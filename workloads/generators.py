"""Generators for BASELINE.json configs 1-5 (BJ:7-11) and scaled variants.

No Krylov arithmetic lives here.  Every generator is deterministic (NumPy
PCG64 with the seeds below, or closed form), so the oracle and the GPU path
see identical bytes.  The recipe of each config is restated in DESIGN.md
§"Input recipe"; the readings of the configs' wording are SURVEY.md §8(c)
Q9-Q11.
"""

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "CONFIGS", "cfg1", "cfg2", "cfg3_rows", "cfg3_rhs", "cfg3", "gauss_shifted_rows",
    "dda_lattice_rows", "dda_lattice_rhs", "cfg2_like", "cfg4_rows", "cfg4_rhs",
    "helmholtz_csr", "helmholtz_rhs", "cfg5", "dense_random", "lattice_dims", "BLOCK",
    "lattice_csr", "helmholtz_coeffs", "dda_kernel", "graded_svd",
]

# config index -> (dtype, n, methods, tol, maxit)  (BJ:7-11, maxit per Q8)
CONFIGS = {
    1: dict(dtype="c128", n=256, methods=("bicgstab", "cgne"), tol=1e-10, maxit=500),
    2: dict(dtype="c128", n=4096, methods=("bicgstab", "qmr", "bicor"), tol=1e-8, maxit=1000),
    3: dict(dtype="c64", n=32768, methods=("bicgstab", "cgne"), tol=1e-5, maxit=500),
    4: dict(dtype="c128", n=65536, methods=("bicgstab",), tol=1e-8, maxit=2000),
    5: dict(dtype="c128", n=128 ** 3, methods=("bicgstab", "cors"), tol=1e-8, maxit=20000),
}


# ---------------------------------------------------------------------------
# cfg1: dense c128 n=256, A = (4+0.5i)I + G/sqrt(n), G parts iid N(0,1), seed 0
# ---------------------------------------------------------------------------
def cfg1(n=256, seed=0):
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    A = G / math.sqrt(n)
    A[np.diag_indices(n)] += (4 + 0.5j)
    y = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / math.sqrt(2)
    return A.astype(np.complex128), y.astype(np.complex128)


# ---------------------------------------------------------------------------
# cfg3: dense c64 n=32768, A = (2+0.3i)I + 0.5 G/sqrt(n), G iid CN(0,1), seed 1.
# Row blocks of BLOCK rows are drawn from independent streams
# default_rng([seed, block]) so any row shard (and any sampled row) can be
# regenerated alone and in parallel.  y comes from default_rng([seed, 2**31]).
# ---------------------------------------------------------------------------
BLOCK = 256


def _gauss_block(n, seed, b, r0, r1, out, shift, scale):
    """Rows [r0, r1) of block b into ``out`` (complex64, shape (r1-r0, n))."""
    rng = np.random.default_rng([seed, b])
    rows = min(BLOCK, n - b * BLOCK)
    re = rng.standard_normal((rows, n), dtype=np.float32)
    im = rng.standard_normal((rows, n), dtype=np.float32)
    lo, hi = r0 - b * BLOCK, r1 - b * BLOCK
    sc = np.float32(scale)
    blk = out
    blk.real[...] = re[lo:hi] * sc
    blk.imag[...] = im[lo:hi] * sc
    for i in range(r0, r1):
        blk[i - r0, i] += np.complex64(shift)


def gauss_shifted_rows(n, r0, r1, seed=1, shift=2 + 0.3j, amp=0.5, out=None, threads=None):
    """Rows [r0, r1) of A = shift·I + amp·G/sqrt(n), G iid CN(0,1) (complex64)."""
    if out is None:
        out = np.empty((r1 - r0, n), dtype=np.complex64)
    scale = amp / math.sqrt(2.0 * n)         # CN(0,1): parts N(0, 1/2)
    jobs = []
    b0, b1 = r0 // BLOCK, (r1 - 1) // BLOCK
    for b in (range(b0, b1 + 1) if r1 > r0 else ()):
        lo = max(r0, b * BLOCK)
        hi = min(r1, (b + 1) * BLOCK)
        jobs.append((b, lo, hi))
    threads = threads or min(len(jobs), os.cpu_count() or 1) or 1

    def work(j):
        b, lo, hi = j
        _gauss_block(n, seed, b, lo, hi, out[lo - r0:hi - r0], shift, scale)

    if threads > 1 and len(jobs) > 1:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, jobs))
    else:
        for j in jobs:
            work(j)
    return out


def cfg3_rhs(n=32768, seed=1):
    rng = np.random.default_rng([seed, 2 ** 31])
    y = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) / math.sqrt(2)
    return y.astype(np.complex64)


def cfg3_rows(r0, r1, n=32768, seed=1, out=None):
    return gauss_shifted_rows(n, r0, r1, seed=seed, out=out)


def cfg3(n=32768, seed=1):
    return cfg3_rows(0, n, n=n, seed=seed), cfg3_rhs(n, seed)


# ---------------------------------------------------------------------------
# cfg2 / cfg4: DDA-like lattice (Q10).  Unit spacing, 0-based integer
# coordinates, x-fastest index j = ix + nx*iy + nx*ny*iz.
# A_ij = 0.1*exp(i*k*d_ij)/d_ij, A_ii = diag, y_j = exp(i*k*z_j).
# ---------------------------------------------------------------------------
def lattice_dims(n_or_dims):
    if isinstance(n_or_dims, tuple):
        return n_or_dims
    return {4096: (16, 16, 16), 65536: (64, 32, 32)}[n_or_dims]


def _coords(nx, ny, nz):
    j = np.arange(nx * ny * nz)
    return j % nx, (j // nx) % ny, j // (nx * ny)


def dda_lattice_rows(dims, k, diag, r0, r1, out=None):
    nx, ny, nz = dims
    n = nx * ny * nz
    ix, iy, iz = _coords(nx, ny, nz)
    if out is None:
        out = np.empty((r1 - r0, n), dtype=np.complex128)
    step = 512
    for a in range(r0, r1, step):
        b = min(r1, a + step)
        dx = (ix[a:b, None] - ix[None, :]).astype(np.float64)
        dy = (iy[a:b, None] - iy[None, :]).astype(np.float64)
        dz = (iz[a:b, None] - iz[None, :]).astype(np.float64)
        d = np.sqrt(dx * dx + dy * dy + dz * dz)
        with np.errstate(divide="ignore", invalid="ignore"):
            blk = 0.1 * np.exp(1j * k * d) / d
        rows = np.arange(a, b)
        blk[rows - a, rows] = diag
        out[a - r0:b - r0] = blk
    return out


def dda_kernel(dims, k, scale=0.1):
    """K(δ) = scale·exp(i k|δ|)/|δ| for every lattice displacement δ (the
    off-diagonal entries of dda_lattice_rows as a 3-level Toeplitz kernel),
    shape (2nz−1, 2ny−1, 2nx−1), index [dz+nz−1, dy+ny−1, dx+nx−1]; δ = 0 → 0.
    Same float64 operations as dda_lattice_rows, so the values agree bitwise."""
    nx, ny, nz = dims
    dz, dy, dx = np.meshgrid(np.arange(-(nz - 1), nz), np.arange(-(ny - 1), ny), np.arange(-(nx - 1), nx),
                             indexing="ij")
    dx, dy, dz = (a.astype(np.float64) for a in (dx, dy, dz))
    d = np.sqrt(dx * dx + dy * dy + dz * dz)
    with np.errstate(divide="ignore", invalid="ignore"):
        K = scale * np.exp(1j * k * d) / d
    K[nz - 1, ny - 1, nx - 1] = 0
    return K.astype(np.complex128)


def dda_lattice_rhs(dims, k):
    nx, ny, nz = dims
    _, _, iz = _coords(nx, ny, nz)
    return np.exp(1j * k * iz.astype(np.float64)).astype(np.complex128)


def cfg2_like(dims=(16, 16, 16), k=1.0, diag=3 + 0.5j):
    n = dims[0] * dims[1] * dims[2]
    return dda_lattice_rows(dims, k, diag, 0, n), dda_lattice_rhs(dims, k)


def cfg2():
    return cfg2_like((16, 16, 16), 1.0, 3 + 0.5j)


def cfg4_rows(r0, r1, out=None):
    return dda_lattice_rows((64, 32, 32), 0.5, 2.5 + 0.2j, r0, r1, out=out)


def cfg4_rhs():
    return dda_lattice_rhs((64, 32, 32), 0.5)


# ---------------------------------------------------------------------------
# cfg5: shifted Helmholtz, 7-point -Δu - (k² + i·0.5·k²)u on an N³ grid,
# h = 1, kh = 10/128, Dirichlet (outside unknowns are 0), x-fastest ordering.
# A_jj = 6 - k²(1 + 0.5i), neighbours -1.  Columns sorted within each row.
# y = 1 at the centre (N/2, N/2, N/2), else 0  (Q11).
# ---------------------------------------------------------------------------
def helmholtz_csr(N=128, kh=10.0 / 128, z0=0, z1=None, dtype=np.complex128):
    """CSR rows of the z-slab [z0, z1) (all rows by default), GLOBAL columns.

    Returns (rowptr int32 local, colind int32 global, vals)."""
    z1 = N if z1 is None else z1
    k2 = kh * kh
    dval = dtype(complex(6.0 - k2, -0.5 * k2))
    r0, r1 = z0 * N * N, z1 * N * N
    j = np.arange(r0, r1, dtype=np.int64)
    ix, iy, iz = j % N, (j // N) % N, j // (N * N)
    offs = (-N * N, -N, -1, 0, 1, N, N * N)
    valid = np.stack([iz > 0, iy > 0, ix > 0, np.ones_like(ix, bool),
                      ix < N - 1, iy < N - 1, iz < N - 1], axis=1)
    cols = j[:, None] + np.array(offs, dtype=np.int64)[None, :]
    vals = np.full(cols.shape, dtype(-1.0), dtype=dtype)
    vals[:, 3] = dval
    counts = valid.sum(axis=1)
    rowptr = np.zeros(r1 - r0 + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    colind = cols[valid].astype(np.int32)
    v = vals[valid]
    return rowptr.astype(np.int32), colind, v


def lattice_csr(nx, ny, nz, d, ox, oy=None, oz=None, z0=0, z1=None, dtype=np.complex128):
    """CSR of the constant-coefficient 7-point operator on an nx × ny × nz
    lattice (x fastest, Dirichlet): diagonal d, x/y/z neighbours ox/oy/oz.
    Rows of the z-slab [z0, z1), GLOBAL columns, sorted.  The stencil
    operator's matrix (ccg_set_matvec_stencil7) written out for the oracle."""
    oy = ox if oy is None else oy
    oz = ox if oz is None else oz
    z1 = nz if z1 is None else z1
    P = nx * ny
    j = np.arange(z0 * P, z1 * P, dtype=np.int64)
    ix, iy, iz = j % nx, (j // nx) % ny, j // P
    offs = (-P, -nx, -1, 0, 1, nx, P)
    valid = np.stack([iz > 0, iy > 0, ix > 0, np.ones_like(ix, bool),
                      ix < nx - 1, iy < ny - 1, iz < nz - 1], axis=1)
    cols = j[:, None] + np.array(offs, dtype=np.int64)[None, :]
    vals = np.empty(cols.shape, dtype=dtype)
    for c, v in enumerate((oz, oy, ox, d, ox, oy, oz)):
        vals[:, c] = dtype(v)
    rowptr = np.zeros(len(j) + 1, dtype=np.int64)
    np.cumsum(valid.sum(axis=1), out=rowptr[1:])
    return rowptr.astype(np.int32), cols[valid].astype(np.int32), vals[valid]


def helmholtz_coeffs(kh=10.0 / 128):
    """(d, o) of config 5's operator (Q11): d = 6 − k²(1 + i/2), o = −1."""
    k2 = kh * kh
    return complex(6.0 - k2, -0.5 * k2), -1.0


def helmholtz_rhs(N=128, z0=0, z1=None, dtype=np.complex128):
    z1 = N if z1 is None else z1
    y = np.zeros((z1 - z0) * N * N, dtype=dtype)
    c = N // 2
    jc = c + N * c + N * N * c
    if z0 * N * N <= jc < z1 * N * N:
        y[jc - z0 * N * N] = 1.0
    return y


def cfg5(N=128):
    rp, ci, v = helmholtz_csr(N)
    return rp, ci, v, helmholtz_rhs(N)


# ---------------------------------------------------------------------------
# small fixtures for parity edge cases
# ---------------------------------------------------------------------------
def dense_random(n, seed=0, dtype=np.complex128, shift=0.0, scale=None):
    """A = shift·I + scale·(G_re + i·G_im), G parts iid N(0,1); default scale 1/sqrt(n)."""
    rng = np.random.default_rng(seed)
    scale = 1.0 / math.sqrt(max(n, 1)) if scale is None else scale
    A = scale * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    A[np.diag_indices(n)] += shift
    return A.astype(dtype)


def graded_svd(n=8, decades=5, seed=5, dtype=np.complex128):
    """SPEC.md:281 (finalize) fixture: a seeded n×n system with singular values
    logspace(0, −decades, n) between two random unitary factors (QR of
    complex Gaussian matrices from default_rng(seed), drawn in the order U, V,
    then y).  Near stagnation at tight tolerances the CGS recurrence residual
    drifts below the attainable true residual (the FALSE_CONVERGENCE case)."""
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    s = np.logspace(0, -float(decades), n)
    A = (U * s) @ V.conj().T
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return A.astype(dtype), y.astype(dtype)
