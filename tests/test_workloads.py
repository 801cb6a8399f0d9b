"""Generators: determinism, shard consistency, closed-form structure (CPU only)."""

import numpy as np

from workloads import (gauss_shifted_rows, cfg3_rhs, helmholtz_csr, helmholtz_rhs,
                       dda_lattice_rows, dda_lattice_rhs, cfg1, cfg2)


def test_gauss_rows_shard_consistency():
    n = 700                                   # ragged last block (BLOCK = 256)
    full = gauss_shifted_rows(n, 0, n, seed=1)
    part = gauss_shifted_rows(n, 300, 517, seed=1)
    np.testing.assert_array_equal(full[300:517], part)
    assert full.dtype == np.complex64
    assert full[5, 5] - full[5, 5].real + full[5, 5].real == full[5, 5]
    # diagonal shift 2+0.3i and off-diagonal scale 0.5/sqrt(n) (CN(0,1) entries)
    off = full[~np.eye(n, dtype=bool)]
    assert abs(np.mean(np.abs(off) ** 2) * n / 0.25 - 1) < 0.01
    assert abs(np.mean(np.diag(full)) - (2 + 0.3j)) < 0.01
    np.testing.assert_array_equal(cfg3_rhs(n), cfg3_rhs(n))


def test_helmholtz_structure():
    N = 128
    rp, ci, v = helmholtz_csr(N, z0=0, z1=2)
    assert rp[-1] == len(ci) == len(v)
    # total nnz of the full 128^3 operator: 7 n - 6 N^2 (closed form) = 14,581,760
    counts = 7 * N ** 3 - 6 * N ** 2
    assert counts == 14_581_760
    # rows sorted by column, global columns, slab rows are contiguous
    for i in (0, 1, 5000, 2 * N * N - 1):
        cols = ci[rp[i]:rp[i + 1]]
        assert np.all(np.diff(cols) > 0)
    y = helmholtz_rhs(N)
    assert y.sum() == 1 and y[64 + 128 * 64 + 128 * 128 * 64] == 1
    # slab decomposition reproduces the whole operator
    rp_a, ci_a, v_a = helmholtz_csr(8)
    parts = [helmholtz_csr(8, z0=z, z1=z + 2) for z in range(0, 8, 2)]
    np.testing.assert_array_equal(np.concatenate([p[1] for p in parts]), ci_a)
    np.testing.assert_array_equal(np.concatenate([p[2] for p in parts]), v_a)


def test_dda_lattice_symmetric_and_rows():
    A, y = cfg2()
    assert A.shape == (4096, 4096)
    np.testing.assert_array_equal(A, A.T)                       # complex symmetric, bitwise
    assert A[0, 0] == 3 + 0.5j
    # A_01: points (0,0,0) and (1,0,0): d = 1
    assert A[0, 1] == 0.1 * np.exp(1j * 1.0) / 1.0
    # A_0,16: (0,1,0): d = 1 ; A_0,17: (1,1,0): d = sqrt 2
    assert np.isclose(A[0, 17], 0.1 * np.exp(1j * np.sqrt(2)) / np.sqrt(2), rtol=1e-15)
    part = dda_lattice_rows((16, 16, 16), 1.0, 3 + 0.5j, 1000, 1100)
    np.testing.assert_array_equal(part, A[1000:1100])
    np.testing.assert_array_equal(y, dda_lattice_rhs((16, 16, 16), 1.0))


def test_cfg1_deterministic():
    A1, y1 = cfg1()
    A2, y2 = cfg1()
    np.testing.assert_array_equal(A1, A2)
    np.testing.assert_array_equal(y1, y2)


def test_lattice_csr_matches_helmholtz_and_closed_form():
    """lattice_csr (the stencil operator written out) equals the config-5
    generator bitwise on a cube, and on a non-cubic lattice its closed-form
    eigenvectors ⊗ sin(π m i/(N+1)) give λ = d + 2 Σ o_a cos(π m_a/(N_a+1))."""
    import numpy as np
    from workloads import lattice_csr, helmholtz_csr, helmholtz_coeffs
    from oracle import CsrOp
    d, o = helmholtz_coeffs()
    for a, b in zip(lattice_csr(9, 9, 9, d, o), helmholtz_csr(9)):
        assert a.dtype == b.dtype and np.array_equal(a, b)
    nx, ny, nz = 7, 5, 4
    ox, oy, oz = -1.0 + 0.1j, -0.5, -2.0j
    op = CsrOp(*lattice_csr(nx, ny, nz, 3 + 1j, ox, oy, oz))
    m = (2, 3, 1)
    vx, vy, vz = (np.sin(np.pi * mm * np.arange(1, N + 1) / (N + 1)) for mm, N in zip(m, (nx, ny, nz)))
    v = np.einsum("k,j,i->kji", vz, vy, vx).ravel().astype(np.complex128)
    lam = (3 + 1j) + 2 * sum(oo * np.cos(np.pi * mm / (N + 1)) for oo, mm, N in zip((ox, oy, oz), m, (nx, ny, nz)))
    assert np.linalg.norm(op.apply(v) - lam * v) <= 1e-13 * np.linalg.norm(v) * abs(lam)
