"""Helpers for the -m gpu parity tests (test infrastructure)."""

import numpy as np
import torch

import paper_1208_4869_b200 as ccg

DEV = "cuda:0"
TOL = {np.complex128: 1e-13, np.complex64: 1e-5}        # per-matvec (north_star)
XTOL = {np.complex128: 1e-9, np.complex64: 1e-4}        # solution (north_star)


def dt_name(dtype):
    return "c64" if np.dtype(dtype) == np.complex64 else "c128"


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def relerr(a, b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


class Dense:
    """A handle over a dense matrix held in a device tensor."""

    def __init__(self, A, lda=None, flags=0):
        A = np.ascontiguousarray(A)
        self.n = A.shape[0]
        self.dtype = A.dtype.type
        if lda is not None and lda != self.n:
            P = np.zeros((self.n, lda), dtype=A.dtype)
            P[:, :self.n] = A
            self.A = to_dev(P)
        else:
            self.A = to_dev(A)
            lda = self.n
        self.h = ccg.ccg_create(dt_name(self.dtype), self.n)
        ccg.ccg_set_matvec_dense(self.h, self.A, 0, self.n, lda=lda, flags=flags)

    def apply(self, x, op="A"):
        xd = to_dev(x.astype(self.dtype))
        y = torch.empty_like(xd)
        ccg.ccg_apply(self.h, op, xd, y)
        return y.cpu().numpy()

    def solve(self, method, y, tol, maxit, x0=None):
        yd = to_dev(y.astype(self.dtype))
        x = torch.empty_like(yd)
        x0d = None if x0 is None else to_dev(x0.astype(self.dtype))
        r = ccg.ccg_solve(self.h, method, x0d, yd, x, tol, maxit)
        r["x"] = x.cpu().numpy()
        r["hist"] = ccg.ccg_get_history(self.h)
        return r

    def close(self):
        ccg.ccg_destroy(self.h)

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Csr(Dense):
    def __init__(self, rowptr, colind, vals, n, flags=0):
        self.n = n
        self.dtype = vals.dtype.type
        self.rp, self.ci, self.v = to_dev(rowptr), to_dev(colind), to_dev(vals)
        self.h = ccg.ccg_create(dt_name(self.dtype), n)
        ccg.ccg_set_matvec_csr(self.h, self.rp, self.ci, self.v, 0, n, len(vals), flags=flags)


def envelope_parity(method, op, y, tol, maxit, dtype, g, solve_at_k, rec=None, **kw):
    """SURVEY §8(c) P-envelope, all four criteria (oracle/envelope.py):
    (1) k_GPU ∈ [k_min − m, k_max + m], m = max(2, ⌈(k_max − k_min)/4⌉)
    (reading E5); (2) x at equal k within max(bar, 2·D)
    with D the pairwise spread; (3) true residual ≤ 10·tol; (4) the GPU
    residual history (g["hist"]) agrees with the clean oracle history to H
    over the envelope's agreement window (where the members agree to H/10).  `g` is the GPU result of the
    tolerance-driven solve; `solve_at_k(k)` returns the GPU x after exactly k
    iterations."""
    from oracle.envelope import envelope, x_spread
    env = envelope(method, op, y, tol, maxit, **kw)
    rec = {} if rec is None else rec
    rec.update(envelope_k=[env.k_min, env.k_max], envelope_window=env.window)
    assert env.check_k(g["iterations"]), rec
    k = min(g["iterations"], env.k_clean)
    xc, D = x_spread(method, op, y, k, **kw)
    err = relerr(solve_at_k(k), xc)
    herr = env.history_error(g["hist"])
    rec.update(envelope_D=D, x_err_equal_k=err, hist_err=herr)
    assert err <= max(XTOL[np.dtype(dtype).type], 2 * D), rec
    assert g["true_rel_res"] <= 10 * tol, rec
    assert herr <= env.H, rec       # over the window where the members agree to H/10 (reading E3)
    return rec
