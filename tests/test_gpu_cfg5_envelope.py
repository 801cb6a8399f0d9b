"""BASELINE config 5 at FULL size (sparse c128 shifted Helmholtz, 128³ CSR,
n = 2,097,152; BJ:11 — the paper's "own sparse matrix scheme" operator,
PAPER.md:95 §5) against the oracle's rounding envelope (SURVEY §8(c)
P-envelope).

The envelope was computed once by `tools/make_cfg5_envelope.py`, which calls
only oracle/ (the clean run and 8 noise seeds take ~1 h of CPU), and stored in
`tests/golden/cfg5_envelope.json`.  Every operator and launch knob the
library has for this problem must land inside it:

  (1) iteration count in [k_min − m, k_max + m], m = max(2, ⌈range/4⌉)
      (oracle/envelope.k_margin, reading E5);
  (4) residual history equal to the clean oracle history to H = 1e-8 over the
      envelope's agreement window (the members agree to H/10 there;
      oracle/envelope.py, reading E3);
  (3) true residual ≤ 10·tol, recomputed here by the oracle's own CSR product;
  (2) x after exactly k iterations within max(1e-9, 2·D(k)) of the clean
      oracle iterate, for the k at which the golden file records D(k) (the
      oracle's clean iterate is recomputed here: ≤ 40 iterations).
"""

import json
import os

import numpy as np
import pytest

import oracle
from oracle import CsrOp
from oracle.envelope import window_from_spread, history_error, WINDOW_FACTOR, k_margin
from workloads import helmholtz_csr, helmholtz_rhs, helmholtz_coeffs
from tests._gpu import Csr, relerr
from tests.test_gpu_next import Stencil
from tests.test_gpu_solve import _record

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cfg5_envelope.json")
N = 128

VARIANTS = [
    ("csr", {}),                              # library SELL-32 copy, one row per step (default)
    ("csr", {"CCG_SELL_ONE": "0"}),           # SELL-32, two rows per step
    ("csr", {"CCG_SPMV": "stream"}),          # CSR-stream blocks
    ("csr", {"CCG_SPMV": "lanes"}),           # 8 lanes per row
    ("stencil", {"CCG_STENCIL_ZC": "4"}),     # matrix-free operator (NEXT-4), z-chunks
    ("stencil", {"CCG_STENCIL_ZC": "8"}),
    ("stencil", {"CCG_STENCIL_ZC": "16"}),
    ("csr", {"CCG_BS_FUSE_RO": "1"}),         # BiCGSTAB's S pass folded into t = A s
    ("stencil", {"CCG_BS_FUSE_RO": "1"}),
]


@pytest.fixture(scope="module")
def problem():
    rp, ci, v = helmholtz_csr(N)
    return rp, ci, v, helmholtz_rhs(N), CsrOp(rp, ci, v), json.load(open(GOLD))


_XC = {}


def _oracle_x(op, y, method, k):
    if (method, k) not in _XC:
        _XC[(method, k)] = oracle.solve(method, op, y, 0.0, k).x
    return _XC[(method, k)]


def _handle(kind, rp, ci, v):
    if kind == "csr":
        return Csr(rp, ci, v, N ** 3)
    d, o = helmholtz_coeffs()
    return Stencil(N, N, N, d, o)


@pytest.mark.parametrize("method", ["bicgstab", "cors"])
@pytest.mark.parametrize("kind,env", VARIANTS, ids=[f"{k}-{'-'.join(f'{a}={b}' for a, b in e.items()) or 'default'}"
                                                     for k, e in VARIANTS])
def test_cfg5_full_size_envelope(problem, method, kind, env, monkeypatch):
    rp, ci, v, y, op, gold = problem
    e = gold["methods"][method]
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    with _handle(kind, rp, ci, v) as h:
        g = h.solve(method, y, gold["tol"], gold["maxit"])
        xk = {int(k): h.solve(method, y, 0.0, int(k))["x"] for k in e["D"]}
    rec = dict(test="cfg5-full-envelope", op=kind, env=env, method=method, status=g["status"],
               k_gpu=g["iterations"], envelope_k=[e["k_min"], e["k_max"]], seeds=e.get("seeds", 8))
    # (4) history over the agreement window (members agree to H/10, reading E3)
    win = window_from_spread(e["hist_spread"], gold["H"] * WINDOW_FACTOR)
    rec["window"] = win
    rec["hist_err"] = history_error(g["hist"], e["hist_clean"], win)
    # (3) true residual by the oracle's CSR product
    tr = np.linalg.norm(y - op.apply(g["x"])) / np.linalg.norm(y)
    rec["true_rel_res"] = tr
    # (2) x at equal k
    xerr = {}
    for k, D in e["D"].items():
        xerr[k] = relerr(xk[int(k)], _oracle_x(op, y, method, int(k)))
        rec[f"x_err_k{k}"] = xerr[k]
    _record(**rec)                     # recorded before the verdict
    assert g["status"] == "CONVERGED", rec
    m = k_margin(e["k_min"], e["k_max"])
    assert e["k_min"] - m <= g["iterations"] <= e["k_max"] + m, rec           # (1)
    assert rec["hist_err"] <= gold["H"], rec                                     # (4)
    assert tr <= 10 * gold["tol"], rec                                           # (3)
    assert abs(tr - g["true_rel_res"]) <= 1e-3 * tr + 1e-15, rec
    for k, D in e["D"].items():                                                  # (2)
        assert xerr[k] <= max(1e-9, 2 * D), rec


# ---------------------------------------------------------------------------
# N = 64 proxy of config 5 (262 144 unknowns, the same k·h = 10/128): the FULL
# P-envelope computed in-test by the oracle (8 noise seeds) —
# k-range, x at equal k against the clean iterate within max(1e-9, 2·D(k)),
# history agreement over the window, true residual — for both operators.
# ---------------------------------------------------------------------------
_ENV64 = {}


def _env64(method):
    from oracle.envelope import envelope, x_spread
    if method not in _ENV64:
        N64 = 64
        rp, ci, v = helmholtz_csr(N64, kh=10 / 128)
        y = helmholtz_rhs(N64)
        op = CsrOp(rp, ci, v)
        env = envelope(method, op, y, 1e-8, 4000)
        xs = {k: x_spread(method, op, y, k) for k in (15, 40)}   # a tight and a loose D(k)
        _ENV64[method] = (rp, ci, v, y, op, env, xs)
    return _ENV64[method]


@pytest.mark.parametrize("kind", ["csr", "stencil"])
@pytest.mark.parametrize("method", ["bicgstab", "cors"])
def test_cfg5_proxy64_full_envelope(method, kind):
    rp, ci, v, y, op, env, xs = _env64(method)
    N64 = 64
    if kind == "csr":
        h = Csr(rp, ci, v, N64 ** 3)
    else:
        d, o = helmholtz_coeffs(10 / 128)
        h = Stencil(N64, N64, N64, d, o)
    with h:
        g = h.solve(method, y, 1e-8, 4000)
        xk = {k: h.solve(method, y, 0.0, k)["x"] for k in xs}
    tr = np.linalg.norm(y - op.apply(g["x"])) / np.linalg.norm(y)
    rec = dict(test="cfg5-proxy64-envelope", op=kind, method=method, k_gpu=g["iterations"],
               envelope_k=[env.k_min, env.k_max], hist_err=env.history_error(g["hist"]), window=env.window,
               true_rel_res=tr)
    for k, (xc, D) in xs.items():
        rec[f"D{k}"], rec[f"x_err{k}"] = D, relerr(xk[k], xc)
    _record(**rec)
    assert g["status"] == "CONVERGED", rec
    assert env.check_k(g["iterations"]), rec                      # (1)
    for k, (xc, D) in xs.items():                                  # (2)
        assert rec[f"x_err{k}"] <= max(1e-9, 2 * D), rec
    assert tr <= 10 * 1e-8, rec                                    # (3)
    assert rec["hist_err"] <= env.H, rec                           # (4)
