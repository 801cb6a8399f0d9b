"""The row-sharded multi-rank path on ONE GPU (loopback communicator).

ccg_create_loopback_group wires G handles (ranks) to an in-process
communicator: the collectives of the NCCL path (allgather of GEMV inputs,
reduce-scatter of Aᴴ partials, allgather of scalar partial sums, CSR halo
exchange) become host barriers + device copies, so the exact sharded code
path — row ownership, slice offsets, halo maps, rank-ordered scalar sums —
runs with the real sm_100a kernels, one host thread per rank, and no kernel
waits on another rank.  Checked against the oracle and the 1-rank result.
"""

import threading

import numpy as np
import pytest

import paper_1208_4869_b200 as ccg
import oracle
from oracle import DenseOp, CsrOp
from oracle.operators import reference_apply
from workloads import cfg1, cfg2, dense_random, helmholtz_csr, helmholtz_rhs
from tests._gpu import to_dev, relerr, XTOL, TOL, Dense, envelope_parity

pytestmark = pytest.mark.gpu


def _threads(G, fn):
    out, errs = [None] * G, []

    def run(r):
        try:
            out[r] = fn(r)
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append((r, e))
    ts = [threading.Thread(target=run, args=(r,)) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    return out


class DenseGroup:
    def __init__(self, A, G, options=0):
        self.n = A.shape[0]
        self.G = G
        self.nloc = self.n // G
        self.dtype = A.dtype.type
        self.dt = "c64" if self.dtype == np.complex64 else "c128"
        self.hs = ccg.ccg_create_loopback_group(G, self.dt, self.n, options=options)
        self.parts = [to_dev(A[r * self.nloc:(r + 1) * self.nloc]) for r in range(G)]
        for r in range(G):
            ccg.ccg_set_matvec_dense(self.hs[r], self.parts[r], r * self.nloc, self.nloc, lda=self.n)

    def _sl(self, v, r):
        return to_dev(np.ascontiguousarray(v[r * self.nloc:(r + 1) * self.nloc]).astype(self.dtype))

    def apply(self, x, op="A"):
        def f(r):
            xd = self._sl(x, r)
            y = xd.clone()
            ccg.ccg_apply(self.hs[r], op, xd, y)
            return y.cpu().numpy()
        return np.concatenate(_threads(self.G, f))

    def solve(self, method, y, tol, maxit):
        def f(r):
            yd = self._sl(y, r)
            x = yd.clone()
            res = ccg.ccg_solve(self.hs[r], method, None, yd, x, tol, maxit)
            res["x"] = x.cpu().numpy()
            res["hist"] = ccg.ccg_get_history(self.hs[r])
            return res
        rs = _threads(self.G, f)
        for k in ("status", "iterations", "matvecs_a", "matvecs_ah", "true_rel_res", "rec_rel_res"):
            assert all(r[k] == rs[0][k] for r in rs), (k, [r[k] for r in rs])   # every rank agrees
        assert all(np.array_equal(r["hist"], rs[0]["hist"]) for r in rs)
        out = dict(rs[0])
        out["x"] = np.concatenate([r["x"] for r in rs])
        return out

    def close(self):
        for h in self.hs:
            ccg.ccg_destroy(h)


class CsrGroup(DenseGroup):
    def __init__(self, N, G, flags=0, options=0):
        self.n = N ** 3
        self.G = G
        self.nloc = self.n // G
        self.dtype = np.complex128
        self.hs = ccg.ccg_create_loopback_group(G, "c128", self.n, options=options)
        zs = N // G
        self.keep = []
        parts = [helmholtz_csr(N, kh=10 / 128, z0=r * zs, z1=(r + 1) * zs) for r in range(G)]

        def f(r):
            rp, ci, v = (to_dev(a) for a in parts[r])
            self.keep.append((rp, ci, v))
            ccg.ccg_set_matvec_csr(self.hs[r], rp, ci, v, r * self.nloc, self.nloc, len(parts[r][2]),
                                   flags=flags)
        _threads(G, f)   # set_matvec_csr agrees on the halo width collectively


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_sharded_dense_apply(G, dtype):
    n = 2048
    A = dense_random(n, seed=G, dtype=dtype, shift=1.5)
    x = (np.random.default_rng(1).standard_normal(n) + 1j).astype(dtype)
    g = DenseGroup(A, G)
    try:
        for op in ("A", "AH", "AT"):
            assert relerr(g.apply(x, op), reference_apply(A, x, op)) <= TOL[dtype], op
    finally:
        g.close()


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("method", ["bicgstab", "cgne", "qmr", "bicor", "cors",
                                    "bicg", "cgs", "cocr", "cgnr", "tfqmr", "gmres", "bicgstabl", "pbicgstab"])
def test_sharded_cfg1_solve(G, method):
    A, y = cfg1()
    if method == "cocr":
        A = (A + A.T) / 2                      # COCR: complex-symmetric A
    g = DenseGroup(A, G)
    try:
        o = oracle.solve(method, DenseOp(A), y, 1e-10, 500)
        r = g.solve(method, y, 1e-10, 500)
        assert r["status"] == "CONVERGED" and abs(r["iterations"] - o.iterations) <= 2
        assert (r["matvecs_a"], r["matvecs_ah"]) == (o.matvecs_a, o.matvecs_ah)
        k = min(r["iterations"], o.iterations)
        re_ = g.solve(method, y, 0.0, k)
        oe = oracle.solve(method, DenseOp(A), y, 0.0, k)
        assert relerr(re_["x"], oe.x) <= XTOL[np.complex128]
        with Dense(A) as h1:                   # and the 1-rank path
            one = h1.solve(method, y, 1e-10, 500)
        assert abs(one["iterations"] - r["iterations"]) <= 2
    finally:
        g.close()


@pytest.mark.parametrize("method", ["bicgstab", "qmr", "bicor"])
def test_sharded_cfg2_solve(method):
    A, y = cfg2()
    g = DenseGroup(A, 2)
    try:
        o = oracle.solve(method, DenseOp(A), y, 1e-8, 1000)
        r = g.solve(method, y, 1e-8, 1000)
        assert r["status"] == "CONVERGED" and abs(r["iterations"] - o.iterations) <= 2
        k = min(r["iterations"], o.iterations)
        assert relerr(g.solve(method, y, 0.0, k)["x"], oracle.solve(method, DenseOp(A), y, 0.0, k).x) <= 1e-9
    finally:
        g.close()


@pytest.mark.parametrize("G", [2, 4])
def test_sharded_csr_apply_and_solve(G):
    N = 16
    g = CsrGroup(N, G)
    rp, ci, v = helmholtz_csr(N, kh=10 / 128)
    op = CsrOp(rp, ci, v)
    try:
        x = np.random.default_rng(3).standard_normal(N ** 3) + 1j
        assert relerr(g.apply(x, "A"), reference_apply(op, x)) <= 1e-13
        y = helmholtz_rhs(N)
        for method in ("bicgstab", "cors"):
            r = g.solve(method, y, 1e-8, 2000)
            assert r["status"] == "CONVERGED" and r["true_rel_res"] <= 1e-7
            envelope_parity(method, op, y, 1e-8, 2000, np.complex128, r,
                            lambda k: g.solve(method, y, 0.0, k)["x"], dict(method=method, G=G))
        # CSR Aᴴ is single-GPU only
        xd = to_dev(x[:g.nloc].astype(np.complex128))
        with pytest.raises(ccg.CcgError) as e:
            ccg.ccg_apply(g.hs[0], "AH", xd, xd.clone())   # refused before any collective
        assert e.value.code == -3
    finally:
        g.close()


class StencilGroup(DenseGroup):
    def __init__(self, nx, ny, nz, G, coeffs, options=0):
        self.n = nx * ny * nz
        self.G = G
        self.nloc = self.n // G
        self.dtype = np.complex128
        self.hs = ccg.ccg_create_loopback_group(G, "c128", self.n, options=options)
        for r in range(G):
            ccg.ccg_set_matvec_stencil7(self.hs[r], nx, ny, nz, *coeffs)


@pytest.mark.parametrize("G", [2, 4])
def test_sharded_stencil_apply_and_solve(G):
    """z-slab sharded matrix-free stencil: halo planes through the loopback
    communicator; all three products and Aᴴ / A-only methods vs the oracle."""
    from workloads import lattice_csr, helmholtz_coeffs
    nx, ny, nz = 20, 12, 16
    co = (5.5 - 0.25j, -1.0 + 0.125j, -0.5, 0.75j)
    op = CsrOp(*lattice_csr(nx, ny, nz, *co))
    x = (np.random.default_rng(2).standard_normal(op.n) + 0.5j).astype(np.complex128)
    g = StencilGroup(nx, ny, nz, G, co)
    try:
        for o in ("A", "AH", "AT"):
            assert relerr(g.apply(x, o), reference_apply(op, x, o)) <= TOL[np.complex128], o
    finally:
        g.close()
    N = 16
    d, oo = helmholtz_coeffs()
    op = CsrOp(*lattice_csr(N, N, N, d, oo))
    y = helmholtz_rhs(N)
    g = StencilGroup(N, N, N, G, (d, oo))
    try:
        for method in ("bicgstab", "cocr", "qmr"):
            r = g.solve(method, y, 1e-8, 3000)
            envelope_parity(method, op, y, 1e-8, 3000, np.complex128, r,
                            lambda k: g.solve(method, y, 0.0, k)["x"], dict(method=method, G=G))
    finally:
        g.close()


@pytest.mark.parametrize("G", [2, 4])
def test_sharded_toeplitz(G):
    """FFT operator with world > 1: gathered input, replicated transform, own rows."""
    from oracle import ToeplitzOp
    from workloads import dda_kernel
    dims = (8, 6, 4)
    K = dda_kernel(dims, 0.9)
    op = ToeplitzOp(K, dims, 2.5 + 0.3j)
    n = 192
    hs = ccg.ccg_create_loopback_group(G, "c128", n)
    g = DenseGroup.__new__(DenseGroup)
    g.n, g.G, g.nloc, g.dtype, g.dt, g.hs = n, G, n // G, np.complex128, "c128", hs
    try:
        for r in range(G):
            ccg.ccg_set_matvec_toeplitz3(hs[r], *dims, K, 2.5 + 0.3j)
        x = (np.random.default_rng(3).standard_normal(n) + 0.25j).astype(np.complex128)
        for o, f in (("A", op.apply), ("AH", op.apply_h), ("AT", op.apply_t)):
            assert relerr(g.apply(x, o), f(x)) <= 1e-13, o
        y = (np.random.default_rng(4).standard_normal(n) + 1j).astype(np.complex128)
        for m in ("bicgstab", "qmr", "cocr"):
            o = oracle.solve(m, op, y, 1e-10, 500)
            r = g.solve(m, y, 1e-10, 500)
            assert r["status"] == "CONVERGED" and abs(r["iterations"] - o.iterations) <= 2, m
            k = min(r["iterations"], o.iterations)
            assert relerr(g.solve(m, y, 0.0, k)["x"], oracle.solve(m, op, y, 0.0, k).x) <= 1e-9, m
    finally:
        g.close()



# ---------------------------------------------------------------------------
# Replicated-vector mode (CCG_OPT_REPLICATED; SURVEY §8(f) NEXT-2 ii): whole
# vectors on every rank, row-sharded operator, one collective per product
# ---------------------------------------------------------------------------
ALL12 = ["bicgstab", "cgne", "qmr", "bicor", "cors", "bicg", "cgs", "cocr", "cgnr", "tfqmr", "gmres", "bicgstabl",
         "pbicgstab"]


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_replicated_dense_apply(G, dtype):
    n = 2048
    A = dense_random(n, seed=G + 7, dtype=dtype, shift=1.5)
    x = (np.random.default_rng(3).standard_normal(n) + 1j).astype(dtype)
    g = DenseGroup(A, G, options=ccg.OPT_REPLICATED)
    try:
        for op in ("A", "AH", "AT"):
            assert relerr(g.apply(x, op), reference_apply(A, x, op)) <= TOL[dtype], op
    finally:
        g.close()


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("method", ALL12)
def test_replicated_cfg1_solve(G, method):
    """Every method on config 1 with replicated vectors: P-literal against the
    oracle, every rank returns the same result (checked by DenseGroup.solve)."""
    A, y = cfg1()
    if method == "cocr":
        A = (A + A.T) / 2
    g = DenseGroup(A, G, options=ccg.OPT_REPLICATED)
    try:
        o = oracle.solve(method, DenseOp(A), y, 1e-10, 500)
        r = g.solve(method, y, 1e-10, 500)
        assert r["status"] == "CONVERGED" and abs(r["iterations"] - o.iterations) <= 2, (r, o.iterations)
        if r["iterations"] == o.iterations:
            assert (r["matvecs_a"], r["matvecs_ah"]) == (o.matvecs_a, o.matvecs_ah)
        k = min(r["iterations"], o.iterations)
        assert relerr(g.solve(method, y, 0.0, k)["x"], oracle.solve(method, DenseOp(A), y, 0.0, k).x) <= 1e-9
    finally:
        g.close()


@pytest.mark.parametrize("G", [2, 4])
def test_replicated_csr_stencil_toeplitz(G):
    """The sparse, matrix-free and lattice operators with replicated vectors
    (no halo exchange: each rank's rows read the whole vector), incl. the Aᴴ
    methods on the complex-symmetric CSR operator, which the row-sharded mode
    cannot run."""
    from workloads import lattice_csr, helmholtz_coeffs, dda_kernel
    from oracle import ToeplitzOp
    N = 16
    d, oo = helmholtz_coeffs()
    op = CsrOp(*lattice_csr(N, N, N, d, oo))
    y = helmholtz_rhs(N)
    x = (np.random.default_rng(5).standard_normal(op.n) + 0.5j).astype(np.complex128)
    for grp in (CsrGroup(N, G, flags=ccg.FLAG_SYMMETRIC, options=ccg.OPT_REPLICATED),
                StencilGroup(N, N, N, G, (d, oo), options=ccg.OPT_REPLICATED)):
        try:
            for o in ("A", "AH", "AT"):
                assert relerr(grp.apply(x, o), reference_apply(op, x, o)) <= 1e-13, o
            for method in ("bicgstab", "qmr", "cocr"):
                r = grp.solve(method, y, 1e-8, 3000)
                envelope_parity(method, op, y, 1e-8, 3000, np.complex128, r,
                                lambda k: grp.solve(method, y, 0.0, k)["x"], dict(method=method, G=G))
        finally:
            grp.close()
    dims = (8, 6, 4)
    K = dda_kernel(dims, 0.9)
    top = ToeplitzOp(K, dims, 2.5 + 0.3j)
    hs = ccg.ccg_create_loopback_group(G, "c128", 192, options=ccg.OPT_REPLICATED)
    g = DenseGroup.__new__(DenseGroup)
    g.n, g.G, g.nloc, g.dtype, g.dt, g.hs = 192, G, 192 // G, np.complex128, "c128", hs
    try:
        for r in range(G):
            ccg.ccg_set_matvec_toeplitz3(hs[r], *dims, K, 2.5 + 0.3j)
        xt = x[:192]
        for o, f in (("A", top.apply), ("AH", top.apply_h), ("AT", top.apply_t)):
            assert relerr(g.apply(xt, o), f(xt)) <= 1e-13, o
        yt = y[:192] + 1.0
        ot = oracle.solve("bicgstab", top, yt, 1e-10, 500)
        rt = g.solve("bicgstab", yt, 1e-10, 500)
        assert rt["status"] == "CONVERGED" and abs(rt["iterations"] - ot.iterations) <= 2
    finally:
        g.close()


@pytest.mark.parametrize("options", [0, 1])
@pytest.mark.parametrize("G", [2, 4])
def test_sharded_jacobi(G, options):
    """Right Jacobi with the row-sharded and the replicated-vector layouts."""
    rng = np.random.default_rng(12)
    n = 256
    d = np.logspace(0, 4, n) * np.exp(1j * rng.uniform(0, 2 * np.pi, n))
    A = (np.diag(d) + 0.3 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n))
    A = A.astype(np.complex128)
    y = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex128)
    g = DenseGroup(A, G, options=options)
    try:
        _threads(G, lambda r: ccg.ccg_set_jacobi(g.hs[r], to_dev(d[r * g.nloc:(r + 1) * g.nloc].copy())))
        for method in ("bicgstab", "qmr", "gmres"):
            o = oracle.solve_jacobi(method, DenseOp(A), d, y, 1e-10, 500)
            r = g.solve(method, y, 1e-10, 500)
            assert r["status"] == "CONVERGED" and abs(r["iterations"] - o.iterations) <= 2, method
            k = min(r["iterations"], o.iterations)
            assert relerr(g.solve(method, y, 0.0, k)["x"],
                          oracle.solve_jacobi(method, DenseOp(A), d, y, 0.0, k).x) <= 1e-9, method
    finally:
        g.close()


# ---------------------------------------------------------------------------
# the gather fused into the product epilogue
# (CCG_OPT_P2P): every rank's mirror buffer written by the product kernel,
# release/acquire flags — on the loopback the peers are the other handles'
# buffers on the same device, and the host barrier of the exchange means no
# kernel waits on another rank's kernel.  The data movement is the same as the
# allgather's, so products and solves are bitwise identical to the plain
# replicated mode.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_p2p_dense_bitwise(G, dtype):
    n = 1024
    A = dense_random(n, seed=11, dtype=dtype, shift=3 - 1j)
    x = (np.random.default_rng(12).standard_normal(n) + 1j).astype(dtype)
    y = (np.random.default_rng(13).standard_normal(n) + 0.5j).astype(dtype)
    ref = DenseGroup(A, G, options=ccg.OPT_REPLICATED)
    p2p = DenseGroup(A, G, options=ccg.OPT_REPLICATED | ccg.OPT_P2P)
    try:
        for o in ("A", "AH", "AT"):
            assert np.array_equal(p2p.apply(x, o), ref.apply(x, o)), o
        tol = 1e-10 if dtype == np.complex128 else 1e-5
        for method in ("bicgstab", "cgne", "qmr", "cocr", "gmres", "cors"):
            a, b = p2p.solve(method, y, tol, 300), ref.solve(method, y, tol, 300)
            assert a["status"] == b["status"] and a["iterations"] == b["iterations"], method
            assert np.array_equal(a["x"], b["x"]), method
        st = ccg.ccg_get_stats(p2p.hs[0])
        assert st["p2p_exchanges"] > 0 and st["replicated"] == 1, st
    finally:
        ref.close()
        p2p.close()


@pytest.mark.parametrize("G", [2, 4])
def test_p2p_csr_stencil_bitwise(G):
    from workloads import lattice_csr, helmholtz_coeffs
    N = 16
    d, oo = helmholtz_coeffs()
    y = helmholtz_rhs(N)
    x = (np.random.default_rng(5).standard_normal(N ** 3) + 0.5j).astype(np.complex128)
    pairs = [(CsrGroup(N, G, flags=ccg.FLAG_SYMMETRIC, options=ccg.OPT_REPLICATED),
              CsrGroup(N, G, flags=ccg.FLAG_SYMMETRIC, options=ccg.OPT_REPLICATED | ccg.OPT_P2P)),
             (StencilGroup(N, N, N, G, (d, oo), options=ccg.OPT_REPLICATED),
              StencilGroup(N, N, N, G, (d, oo), options=ccg.OPT_REPLICATED | ccg.OPT_P2P))]
    for ref, p2p in pairs:
        try:
            for o in ("A", "AH", "AT"):
                assert np.array_equal(p2p.apply(x, o), ref.apply(x, o)), o
            for method in ("bicgstab", "qmr", "cocr"):
                a, b = p2p.solve(method, y, 1e-8, 3000), ref.solve(method, y, 1e-8, 3000)
                assert a["iterations"] == b["iterations"] and np.array_equal(a["x"], b["x"]), method
        finally:
            ref.close()
            p2p.close()


def test_p2p_option_errors():
    with pytest.raises(ccg.CcgError) as e:           # needs replicated vectors
        ccg.ccg_create_loopback_group(2, "c128", 64, options=ccg.OPT_P2P)
    assert e.value.code == -1
    with pytest.raises(ccg.CcgError) as e:           # at most 8 ranks (one NVLink domain)
        ccg.ccg_create_loopback_group(16, "c128", 64, options=ccg.OPT_P2P | ccg.OPT_REPLICATED)
    assert e.value.code == -1
