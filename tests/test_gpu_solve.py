"""Solver parity: ccg_solve (C-ABI, sm_100a) vs the oracle recurrences.

Bar (north_star): iteration counts within ±2 of the oracle; x compared at an
EQUAL iteration count (stopping one iteration apart moves x by
more than the bar) within 1e-9 (c128) / 1e-4 (c64) relative; true residual
≤ 10·tol.  Plus the method's degenerate cases.
"""

import json
import os

import numpy as np
import pytest

import paper_1208_4869_b200 as ccg
import oracle
from oracle import DenseOp, CsrOp
from workloads import cfg1, cfg2, gauss_shifted_rows, cfg3_rhs, helmholtz_csr, helmholtz_rhs, dense_random
from tests._gpu import Dense, Csr, XTOL, relerr, envelope_parity

pytestmark = pytest.mark.gpu

HOT = ("bicgstab", "cgne", "qmr", "bicor", "cors")


def _record(**kw):
    path = os.environ.get("CCG_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(kw) + "\n")


def _parity(h, op, y, method, tol, maxit, dtype, literal=True, tag=""):
    """P-literal (north_star) and, where a config/method pair is not one
    BASELINE.json names, the P-envelope fallback of SURVEY §8(c) (all four
    criteria, tests/_gpu.envelope_parity)."""
    o = oracle.solve(method, op, y, tol, maxit)
    g = h.solve(method, y, tol, maxit)
    assert g["status"] == o.status_name == "CONVERGED", (method, g["status"], o.status_name)
    assert g["true_rel_res"] <= 10 * tol
    k = min(g["iterations"], o.iterations)
    oe = oracle.solve(method, op, y, 0.0, k)
    ge = h.solve(method, y, 0.0, k)
    assert ge["iterations"] == oe.iterations == k
    err = relerr(ge["x"], oe.x)
    lit = abs(g["iterations"] - o.iterations) <= 2 and err <= XTOL[dtype]
    rec = dict(test=tag, method=method, k_gpu=g["iterations"], k_oracle=o.iterations,
               x_err_equal_k=err, literal=lit)
    if not lit:
        assert not literal, rec
        envelope_parity(method, op, y, tol, maxit, dtype, g, lambda kk: h.solve(method, y, 0.0, kk)["x"], rec)
    _record(**rec)
    return o, g


@pytest.mark.parametrize("method", HOT)
def test_cfg1_all_methods(method):
    A, y = cfg1()
    with Dense(A) as h:
        o, g = _parity(h, DenseOp(A), y, method, 1e-10, 500, np.complex128, tag="cfg1")
        assert (g["matvecs_a"], g["matvecs_ah"]) == (o.matvecs_a, o.matvecs_ah)
        assert g["half_step"] == o.half_step
        h.solve(method, y, 1e-10, 500)          # history of the tolerance-driven solve
        hist = ccg.ccg_get_history(h.h)
        r0 = o.history[0]
        np.testing.assert_allclose(hist, np.array(o.history, float) / r0, rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("method", HOT)
def test_cfg2_all_methods(method):
    A, y = cfg2()
    with Dense(A) as h:
        _parity(h, DenseOp(A), y, method, 1e-8, 1000, np.complex128, tag="cfg2",
                literal=method in ("bicgstab", "qmr", "bicor"))


@pytest.mark.parametrize("method", ["bicgstab", "cgne", "qmr", "bicor", "cors"])
def test_cfg3_proxy_c64(method):
    n = 4096                     # cfg3 recipe at a size the oracle finishes quickly
    A = gauss_shifted_rows(n, 0, n, seed=1)
    y = cfg3_rhs(n)
    with Dense(A) as h:
        _parity(h, DenseOp(A), y, method, 1e-5, 500, np.complex64, tag="cfg3-proxy",
                literal=method in ("bicgstab", "cgne"))


@pytest.mark.parametrize("method", ["bicgstab", "cors"])
def test_cfg5_proxy_csr(method):
    N = 24
    rp, ci, v = helmholtz_csr(N, kh=10 / 128)
    y = helmholtz_rhs(N)
    with Csr(rp, ci, v, N ** 3) as h:
        _parity(h, CsrOp(rp, ci, v), y, method, 1e-8, 2000, np.complex128, literal=False,
                tag="cfg5-proxy")


@pytest.mark.parametrize("n", [1, 7, 257, 1000])
@pytest.mark.parametrize("method", HOT)
def test_ragged_sizes(method, n):
    A = dense_random(n, seed=n, dtype=np.complex128, shift=3 - 1j)
    y = dense_random(n, seed=n + 1)[:, 0] * 3
    with Dense(A) as h:
        _parity(h, DenseOp(A), y, method, 1e-10, 400, np.complex128, tag=f"ragged{n}")


@pytest.mark.parametrize("method", HOT)
def test_scaled_identity(method):
    c = 3 - 4j
    n = 10
    y = np.arange(n) + 1j * np.arange(n)[::-1]
    with Dense(c * np.eye(n, dtype=np.complex128)) as h:
        g = h.solve(method, y.astype(np.complex128), 1e-12, 50)
    assert g["status"] == "CONVERGED" and g["iterations"] == 1
    np.testing.assert_allclose(g["x"], y / c, rtol=1e-14, atol=1e-14)
    if method == "bicgstab":
        assert g["half_step"] and g["matvecs_a"] == 1


def test_breakdown_fixture():
    A = np.array([[0, 1], [-1, 0]], dtype=np.complex128)
    y = np.array([1, 0], dtype=np.complex128)
    with Dense(A) as h:
        g = h.solve("bicgstab", y, 1e-10, 10)
        assert g["status"] == "BREAKDOWN" and g["breakdown"] == "sigma" and g["iterations"] == 0
        for m in ("bicor", "cors"):
            g = h.solve(m, y, 1e-10, 10)
            assert g["status"] == "BREAKDOWN" and g["breakdown"] == "rho", m


@pytest.mark.parametrize("method", HOT)
def test_zero_rhs_maxit_nonfinite_x0(method):
    A, y = cfg1(n=32, seed=2)
    with Dense(A) as h:
        g = h.solve(method, np.zeros(32, np.complex128), 1e-10, 10)
        assert g["status"] == "CONVERGED" and g["iterations"] == 0 and not np.any(g["x"])
        g = h.solve(method, y, 0.0, 3)
        o = oracle.solve(method, DenseOp(A), y, 0.0, 3)
        assert g["status"] == "MAXIT" and g["iterations"] == 3
        assert (g["matvecs_a"], g["matvecs_ah"]) == (o.matvecs_a, o.matvecs_ah)
        yb = y.copy()
        yb[5] = np.nan
        assert h.solve(method, yb, 1e-10, 10)["status"] == "NONFINITE"
        xs = np.linalg.solve(A, y)
        o = oracle.solve(method, DenseOp(A), y, 1e-12, 100, x0=0.5 * xs)
        g = h.solve(method, y, 1e-12, 100, x0=0.5 * xs)
        assert abs(g["iterations"] - o.iterations) <= 2 and relerr(g["x"], o.x) <= 1e-9


def test_capability_and_state_errors():
    rp, ci, v = helmholtz_csr(6)
    with Csr(rp, ci, v, 216) as h:
        for m in ("cgne", "qmr", "bicor"):
            with pytest.raises(ccg.CcgError) as e:
                h.solve(m, np.ones(216, np.complex128), 1e-8, 10)
            assert e.value.code == -3
    h = ccg.ccg_create("c64", 8)
    try:
        with pytest.raises(ccg.CcgError) as e:
            ccg.ccg_solve(h, "bicgstab", None, np.ones(8, np.complex64), np.empty(8, np.complex64), 1e-5, 10)
        assert e.value.code == -4
    finally:
        ccg.ccg_destroy(h)


def test_csr_symmetric_ah_methods():
    """Complex-symmetric CSR with CCG_FLAG_SYMMETRIC runs the Aᴴ methods (single GPU)."""
    N = 10
    rp, ci, v = helmholtz_csr(N, kh=10 / 128)
    y = helmholtz_rhs(N)
    with Csr(rp, ci, v, N ** 3, flags=ccg.FLAG_SYMMETRIC) as h:
        for m in ("cgne", "qmr", "bicor"):
            _parity(h, CsrOp(rp, ci, v), y, m, 1e-8, 3000, np.complex128, literal=False,
                    tag="csr-sym")


def test_host_pointer_solve_and_determinism():
    A, y = cfg2()
    with Dense(A) as h:
        x1 = np.empty(4096, np.complex128)
        r1 = ccg.ccg_solve(h.h, "bicgstab", None, y, x1, 1e-8, 1000)
        r2 = h.solve("bicgstab", y, 1e-8, 1000)
        assert r1["iterations"] == r2["iterations"]
        assert np.array_equal(x1, r2["x"])        # bitwise run-to-run determinism


@pytest.mark.parametrize("method", ["bicgstab", "cgne"])
def test_full_size_cfg3(method):
    """cfg3 at full size (n = 32768 c64, 8.6 GB): literal parity vs the oracle."""
    import torch
    n = 32768
    A = gauss_shifted_rows(n, 0, n, seed=1)
    y = cfg3_rhs(n)
    Ad = torch.from_numpy(A).to("cuda:0")
    h = ccg.ccg_create("c64", n)
    try:
        ccg.ccg_set_matvec_dense(h, Ad, 0, n)
        op = DenseOp(A)

        class H:
            def solve(self, m, yy, tol, maxit):
                yd = torch.from_numpy(yy).to("cuda:0")
                x = torch.empty_like(yd)
                r = ccg.ccg_solve(h, m, None, yd, x, tol, maxit)
                r["x"] = x.cpu().numpy()
                return r
        _parity(H(), op, y, method, 1e-5, 500, np.complex64, tag="cfg3-full")
    finally:
        ccg.ccg_destroy(h)
        del Ad


@pytest.mark.parametrize("method", ["bicgstab", "cors"])
def test_full_size_cfg5_residual_property(method):
    """cfg5 at full size: x from the GPU satisfies ‖y − A x‖ ≤ 10·tol·‖y‖ when
    the residual is recomputed by the oracle's own CSR product (a property
    that holds at any size; literal iterate parity is not attainable on this
    rounding-chaotic indefinite problem)."""
    rp, ci, v = helmholtz_csr(128)
    y = helmholtz_rhs(128)
    n = 128 ** 3
    with Csr(rp, ci, v, n) as h:
        g = h.solve(method, y, 1e-8, 20000)
    assert g["status"] == "CONVERGED"
    op = CsrOp(rp, ci, v)
    tr = np.linalg.norm(y - op.apply(g["x"])) / np.linalg.norm(y)
    assert tr <= 1e-7
    assert abs(tr - g["true_rel_res"]) <= 1e-3 * tr + 1e-15
    _record(test="cfg5-full", method=method, k_gpu=g["iterations"], true_rel_res=tr)


def test_cfg4_device_generator_matches_numpy():
    """Config 4's 68.7 GB matrix is generated on the GPU (workloads/device.py, the
    same closed form as the NumPy generator): sampled row blocks agree with the
    NumPy rows to a few ulp."""
    import torch
    from workloads import cfg4_rows
    from workloads.device import cfg4_rows_device
    for r0 in (0, 4096, 33000, 65536 - 64):
        out = torch.empty((64, 65536), dtype=torch.complex128, device="cuda:0")
        cfg4_rows_device(r0, r0 + 64, out)
        ref = cfg4_rows(r0, r0 + 64)
        got = out.cpu().numpy()
        assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)) <= 4 * np.finfo(float).eps


@pytest.mark.parametrize("flags", [0, ccg.FLAG_SYMMETRIC], ids=["full", "sym"])
def test_cfg4_dense_full_size(flags):
    """BASELINE config 4 at its full size as a DENSE matrix (n = 65536 c128,
    68.7 GB in HBM, the bench_all launch configuration): sampled rows of A·x
    against the oracle's own rows, Aᴴ·x against the oracle's lattice operator,
    and BiCGSTAB inside the rounding envelope of SURVEY §8(c) — the problem is
    rounding-chaotic (noise-seed iteration counts 102-110), so the P-envelope
    criterion applies: k within [k_min − 2, k_max + 2], x at equal k within
    max(1e-9, 2D), and the true residual recomputed by the oracle ≤ 10·tol.
    `sym`: the same with CCG_FLAG_SYMMETRIC (A = Aᵀ bitwise):
    the products read only the upper triangle (matvec.cuh gemv_sym)."""
    import torch
    from oracle import ToeplitzOp
    from oracle.operators import reference_apply
    from workloads import dda_kernel, cfg4_rows, cfg4_rhs
    from workloads.device import cfg4_rows_device
    n = 65536
    dims = (64, 32, 32)
    Ad = torch.empty((n, n), dtype=torch.complex128, device="cuda:0")
    for r0 in range(0, n, 4096):
        cfg4_rows_device(r0, r0 + 4096, Ad[r0:r0 + 4096])
    torch.cuda.synchronize()
    op = ToeplitzOp(dda_kernel(dims, 0.5), dims, 2.5 + 0.2j)
    y = cfg4_rhs()
    h = ccg.ccg_create("c128", n)
    try:
        ccg.ccg_set_matvec_dense(h, Ad, 0, n, flags=flags)
        rng = np.random.default_rng(9)
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        xd = torch.from_numpy(x).to("cuda:0")
        yd = torch.empty_like(xd)
        ccg.ccg_apply(h, "A", xd, yd)
        ax = yd.cpu().numpy()
        for r in (0, 1, 12345, 40000, 65535):
            row = cfg4_rows(r, r + 1)
            assert abs(ax[r] - reference_apply(row, x)[0]) <= 1e-13 * (np.abs(row[0]) @ np.abs(x)), r
        assert relerr(ax, op.apply(x)) <= 1e-13
        ccg.ccg_apply(h, "AH", xd, yd)
        assert relerr(yd.cpu().numpy(), op.apply_h(x)) <= 1e-13

        yv = torch.from_numpy(y).to("cuda:0")
        xo = torch.empty_like(yv)
        g = ccg.ccg_solve(h, "bicgstab", None, yv, xo, 1e-8, 2000)
        g["hist"] = ccg.ccg_get_history(h)
        assert g["status"] == "CONVERGED"
        xg = xo.cpu().numpy()
        tr = np.linalg.norm(y - op.apply(xg)) / np.linalg.norm(y)
        assert tr <= 1e-7

        def at_k(k):
            ccg.ccg_solve(h, "bicgstab", None, yv, xo, 0.0, k)
            return xo.cpu().numpy()
        rec = dict(test="cfg4-full-dense" + ("-sym" if flags else ""), method="bicgstab", k_gpu=g["iterations"],
                   true_rel_res=tr)
        envelope_parity("bicgstab", op, y, 1e-8, 2000, np.complex128, g, at_k, rec)
        _record(**rec)
    finally:
        ccg.ccg_destroy(h)
        del Ad
        torch.cuda.empty_cache()


# ---------------------------------------------------------------------------
# FALSE_CONVERGENCE: the recurrence residual claims
# convergence, the true residual recomputed at exit is > 10·tol
# ---------------------------------------------------------------------------
_FC = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "false_convergence.json")))


def test_false_convergence_spec_fixture():
    """SPEC.md:281's fixture: seeded 8×8 graded system, CGS at tol 1e-15."""
    from workloads import graded_svd
    g = _FC["spec_fixture"]
    A, y = graded_svd(n=8, decades=5, seed=5)
    o = oracle.solve(g["method"], DenseOp(A), y, g["tol"], g["maxit"])
    with Dense(A) as h:
        r = h.solve(g["method"], y, g["tol"], g["maxit"])
    assert o.status_name == r["status"] == g["status"], (o.status_name, r)
    true = np.linalg.norm(y - A @ r["x"]) / np.linalg.norm(y)
    assert r["rec_rel_res"] <= g["tol"] and true > 10 * g["tol"]
    assert r["true_rel_res"] == pytest.approx(true, rel=1e-3)
    _record(test="false-conv-spec", k_gpu=r["iterations"], k_oracle=o.iterations, true_rel_res=true)


@pytest.mark.parametrize("op", ["dense", "csr"])
@pytest.mark.parametrize("method", _FC["single_precision"]["methods"])
def test_false_convergence_single_precision(method, op):
    if op == "csr" and method in ("bicor", "cgne"):
        pytest.skip("Aᴴ methods need CCG_FLAG_SYMMETRIC on CSR; this matrix is not symmetric")
    """c64 working precision at tol 1e-10: the true residual floor (~1e-7) is
    far above 10·tol while the recurrence residual keeps falling."""
    g = _FC["single_precision"]
    n = 256
    A = gauss_shifted_rows(n, 0, n, seed=1)
    y = cfg3_rhs(n)
    o = oracle.solve(method, DenseOp(A), y, g["tol"], g["maxit"])
    if op == "dense":
        h = Dense(A)
    else:
        import scipy.sparse as sp
        M = sp.csr_matrix(A)
        h = Csr(M.indptr.astype(np.int32), M.indices.astype(np.int32), M.data.astype(np.complex64), n)
    with h:
        r = h.solve(method, y, g["tol"], g["maxit"])
    assert r["status"] == o.status_name == g["status"], (method, r["status"], o.status_name)
    assert abs(r["iterations"] - o.iterations) <= 2
    true = np.linalg.norm(y.astype(complex) - A.astype(complex) @ r["x"].astype(complex)) / np.linalg.norm(y)
    assert true > 10 * g["tol"] and r["rec_rel_res"] <= g["tol"]
