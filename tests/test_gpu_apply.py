"""Per-matvec parity: libccg (C-ABI, sm_100a kernels) vs oracle.reference_apply.

Bar (north_star): relative error ≤ 1e-13 (c128) / 1e-5 (c64), normwise, and
componentwise |Δ_i| ≤ tol·(|A||x|)_i.  Sizes span several tiles and ragged
tails (non-powers of two), odd leading dimensions (the unvectorised path),
padded lda, CSR, and the full-size configs in the launch configuration
bench.py uses (sampled rows for A·x; streamed blocks for Aᴴ·x).
"""

import numpy as np
import pytest
import torch

import paper_1208_4869_b200 as ccg
from oracle.operators import reference_apply, CsrOp
from workloads import (dense_random, cfg1, cfg2, gauss_shifted_rows, cfg3_rhs, helmholtz_csr,
                       BLOCK)
from tests._gpu import Dense, Csr, TOL, relerr, to_dev

pytestmark = pytest.mark.gpu


def _x(n, dtype, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(dtype)


def _componentwise_ok(A, x, y_gpu, y_ref, op, tol):
    M = np.abs(A.astype(np.complex128))
    if op != "A":
        M = M.T
    bound = M @ np.abs(x.astype(np.complex128))
    return np.all(np.abs(y_gpu - y_ref) <= 8 * tol * bound + 1e-300)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("n", [1, 2, 3, 31, 64, 257, 1000, 2049, 4097])
@pytest.mark.parametrize("op", ["A", "AH", "AT"])
def test_dense_apply_parity(dtype, n, op):
    A = dense_random(n, seed=n, dtype=dtype, shift=1.0 + 0.5j)
    x = _x(n, dtype, seed=n + 1)
    with Dense(A) as h:
        y = h.apply(x, op)
    ref = reference_apply(A, x, op)
    assert relerr(y, ref) <= TOL[dtype], (n, op)
    assert _componentwise_ok(A, x, y, ref, op, TOL[dtype] * 10)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
@pytest.mark.parametrize("lda", [301, 320])
def test_dense_apply_padded_lda(dtype, lda):
    n = 300
    A = dense_random(n, seed=7, dtype=dtype, shift=2.0)
    x = _x(n, dtype, seed=8)
    with Dense(A, lda=lda) as h:
        for op in ("A", "AH", "AT"):
            assert relerr(h.apply(x, op), reference_apply(A, x, op)) <= TOL[dtype], (lda, op)


@pytest.mark.parametrize("cfg", [1, 2])
def test_config_shapes(cfg):
    A, y = cfg1() if cfg == 1 else cfg2()
    with Dense(A) as h:
        for op in ("A", "AH", "AT"):
            assert relerr(h.apply(y, op), reference_apply(A, y, op)) <= 1e-13


def test_determinism_bitwise():
    A = dense_random(3000, seed=3, dtype=np.complex64, shift=1.0)
    x = _x(3000, np.complex64)
    with Dense(A) as h:
        for op in ("A", "AH"):
            a, b = h.apply(x, op), h.apply(x, op)
            assert np.array_equal(a, b), op


def test_adjoint_identity_on_gpu():
    n = 2000
    A = dense_random(n, seed=9, dtype=np.complex128, shift=0.5)
    x, z = _x(n, np.complex128, 1), _x(n, np.complex128, 2)
    with Dense(A) as h:
        lhs = np.vdot(z, h.apply(x, "A"))
        rhs = np.vdot(h.apply(z, "AH"), x)
        assert abs(lhs - rhs) <= 8 * np.finfo(float).eps * n * np.abs(A).max() * np.linalg.norm(x) * np.linalg.norm(z)
        assert abs(np.dot(z, h.apply(x, "A")) - np.dot(h.apply(z, "AT"), x)) <= 1e-9 * abs(lhs)


def test_host_pointers():
    """ccg_apply accepts host (numpy) vectors: staged by the library."""
    n = 513
    A = dense_random(n, seed=5, dtype=np.complex128)
    x = _x(n, np.complex128, 3)
    with Dense(A) as h:
        y = np.empty(n, np.complex128)
        ccg.ccg_apply(h.h, "A", x, y)
        assert relerr(y, reference_apply(A, x)) <= 1e-13


@pytest.mark.parametrize("N", [5, 16, 33])
def test_csr_apply_parity(N):
    rp, ci, v = helmholtz_csr(N, kh=10 / 128)
    op = CsrOp(rp, ci, v)
    x = _x(op.n, np.complex128, N)
    with Csr(rp, ci, v, op.n, flags=ccg.FLAG_SYMMETRIC) as h:
        for o in ("A", "AH", "AT"):
            assert relerr(h.apply(x, o), reference_apply(op, x, o)) <= 1e-13, o


def test_csr_capability_error():
    rp, ci, v = helmholtz_csr(6)
    with Csr(rp, ci, v, 216) as h:
        with pytest.raises(ccg.CcgError) as e:
            h.apply(_x(216, np.complex128), "AH")
        assert e.value.code == -3


def test_state_error_before_operator():
    h = ccg.ccg_create("c128", 8)
    try:
        x = to_dev(np.ones(8, np.complex128))
        with pytest.raises(ccg.CcgError) as e:
            ccg.ccg_apply(h, "A", x, torch.empty_like(x))
        assert e.value.code == -4
    finally:
        ccg.ccg_destroy(h)


def test_full_size_cfg3_sampled_rows_and_adjoint():
    """cfg3 at its full size (n = 32768 c64, 8.6 GB), bench launch configuration."""
    n = 32768
    Ad = torch.empty((n, n), dtype=torch.complex64, device="cuda")
    host = torch.empty((4096, n), dtype=torch.complex64).pin_memory()
    for r0 in range(0, n, 4096):
        gauss_shifted_rows(n, r0, r0 + 4096, seed=1, out=host.numpy())
        Ad[r0:r0 + 4096].copy_(host, non_blocking=False)
    x = cfg3_rhs(n)
    h = ccg.ccg_create("c64", n)
    try:
        ccg.ccg_set_matvec_dense(h, Ad, 0, n)
        xd = to_dev(x)
        y = torch.empty_like(xd)
        ccg.ccg_apply(h, "A", xd, y)
        y = y.cpu().numpy()
        rows = [0, 1, 255, 256, 4097, 12345, 32767]
        for b in sorted({r // BLOCK for r in rows}):
            blk = gauss_shifted_rows(n, b * BLOCK, (b + 1) * BLOCK, seed=1)
            for r in rows:
                if r // BLOCK == b:
                    ref = reference_apply(blk[r - b * BLOCK][None, :], x)[0]
                    scale = np.abs(blk[r - b * BLOCK]) @ np.abs(x)
                    assert abs(y[r] - ref) <= 1e-5 * scale, r
        # Aᴴx over all rows, streamed from the generator block by block
        yh = torch.empty_like(xd)
        ccg.ccg_apply(h, "AH", xd, yh)
        ref = np.zeros(n, np.complex128)
        for r0 in range(0, n, 4096):
            blk = gauss_shifted_rows(n, r0, r0 + 4096, seed=1)
            ref += reference_apply(blk, x[r0:r0 + 4096], "AH")
        assert relerr(yh.cpu().numpy(), ref) <= 1e-5
    finally:
        ccg.ccg_destroy(h)
        del Ad


def test_full_size_cfg5_apply():
    rp, ci, v = helmholtz_csr(128)
    n = 128 ** 3
    x = _x(n, np.complex128, 11)
    op = CsrOp(rp, ci, v)
    with Csr(rp, ci, v, n) as h:
        y = h.apply(x, "A")
    assert relerr(y, reference_apply(op, x)) <= 1e-13
