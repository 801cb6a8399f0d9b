"""Pins for oracle/envelope.py (the P-envelope of SURVEY §8(c)) and for the
FALSE_CONVERGENCE guard of the oracle's finalize step.

The envelope is part of the parity machinery: every GPU verdict on a
rounding-chaotic config/method pair rests on it.  It is pinned here by what
its definition fixes, independently of its own code:

* the measured noise amplitude of NoisyOp (2e-16 relative per
  matvec output, ξ_re, ξ_im iid N(0,1));
* linear response: D grows in proportion to the noise amplitude;
* D is PAIRWISE: strictly larger than the largest distance from the clean run;
* collapse on a well-conditioned problem (config 1: every member stops at the
  same k, D at rounding level, the agreement window spans the whole history);
* the agreement window of a chaotic problem ends where the member histories
  first split by more than H, and shrinks when the noise grows.
"""

import json
import os

import numpy as np
import pytest

import oracle
from oracle import DenseOp, CsrOp
from oracle.envelope import (NoisyOp, envelope, x_spread, agreement_window, rel_history,
                             pairwise_spread, noise_amplitude)
from oracle.solvers import _finish, _Ctx, Result, CONVERGED, FALSE_CONVERGENCE, MAXIT
from workloads import cfg1, helmholtz_csr, helmholtz_rhs, graded_svd, gauss_shifted_rows, cfg3_rhs, \
    dda_lattice_rows, dda_lattice_rhs

GOLD = os.path.join(os.path.dirname(__file__), "golden", "false_convergence.json")


class _Ident:
    def __init__(self, n, dtype):
        self.n, self.dtype = n, dtype
        self.n_a = self.n_ah = 0

    def apply(self, x):
        return x.copy()

    apply_h = apply_t = apply

    def reset_counts(self):
        pass


# ---------------- noise amplitude ----------------
def test_noise_amplitude_c128_measured():
    """SURVEY §8(c) emulation 2: outputs × (1 + 2e-16·(ξ_re + iξ_im))."""
    n = 400_000
    d = NoisyOp(_Ident(n, np.complex128), seed=1).perturbation(n)
    for part in (d.real, d.imag):
        assert abs(np.mean(part)) < 0.01 * 2e-16
        assert abs(np.std(part) / 2e-16 - 1.0) < 0.01      # ×10 or ×2 fails
    # apply() multiplies every output by exactly these factors (then rounds)
    v = np.random.default_rng(0).standard_normal(n) + 1j
    out = NoisyOp(_Ident(n, np.complex128), seed=1).apply(v)
    assert np.array_equal(out, v + v * d)


def test_noise_amplitude_c64_measured():
    """E1: c64 amplitude = 2e-16 · (2⁻²⁴ / 2⁻⁵³) = 1.07e-7 (the default for a
    complex64 operator)."""
    assert abs(noise_amplitude(np.complex64) / (2e-16 * 2.0 ** 29) - 1) < 1e-12
    n = 400_000
    d = NoisyOp(_Ident(n, np.complex64), seed=2).perturbation(n)
    assert abs(np.std(d.real) / 1.0737e-7 - 1.0) < 0.01


def test_noise_independent_per_product_and_seed():
    op1 = NoisyOp(_Ident(1000, np.complex128), seed=1)
    a, b = op1.apply(np.ones(1000, complex)), op1.apply(np.ones(1000, complex))
    c = NoisyOp(_Ident(1000, np.complex128), seed=2).apply(np.ones(1000, complex))
    assert not np.array_equal(a, b) and not np.array_equal(a, c)
    again = NoisyOp(_Ident(1000, np.complex128), seed=1).apply(np.ones(1000, complex))
    assert np.array_equal(a, again)     # seeded: reproducible


# ---------------- D: linear response, pairwise ----------------
def _lattice_small():
    dims = (6, 6, 6)
    A = dda_lattice_rows(dims, 1.0, 3 + 0.5j, 0, 216)
    return DenseOp(A), dda_lattice_rhs(dims, 1.0)


def test_D_linear_in_noise_amplitude():
    op, y = _lattice_small()
    k = 12
    _, D1 = x_spread("bicgstab", op, y, k, eps=2e-16)
    _, D10 = x_spread("bicgstab", op, y, k, eps=2e-15)
    assert D1 > 0
    assert 6.0 < D10 / D1 < 15.0, (D1, D10)


def test_D_is_pairwise():
    op, y = _lattice_small()
    k = 12
    xs = [oracle.solve("bicgstab", op, y, 0.0, k).x] + \
         [oracle.solve("bicgstab", NoisyOp(op, s), y, 0.0, k).x for s in range(1, 9)]
    nc = np.linalg.norm(xs[0])
    clean_rel = max(np.linalg.norm(x - xs[0]) / nc for x in xs[1:])
    xc, D = x_spread("bicgstab", op, y, k)
    assert np.array_equal(xc, xs[0])
    brute = max(np.linalg.norm(xs[a] - xs[b]) / nc for a in range(9) for b in range(a + 1, 9))
    assert D == pytest.approx(brute, rel=1e-12)
    assert D >= 1.1 * clean_rel              # a clean-relative D would fail this
    assert D <= 2.0 * clean_rel + 1e-300     # triangle inequality through the clean run


def test_pairwise_spread_small():
    xs = [np.array([1.0, 0]), np.array([1.0, 1e-3]), np.array([1.0, -2e-3])]
    assert pairwise_spread(xs, xs[0]) == pytest.approx(3e-3)


# ---------------- collapse on a well-conditioned case ----------------
def test_envelope_collapses_on_cfg1():
    A, y = cfg1()
    op = DenseOp(A)
    e = envelope("bicgstab", op, y, 1e-10, 500)
    assert e.k_min == e.k_max == e.k_clean == 12
    assert e.window == len(e.hist_clean) - 1          # histories agree to 1e-9 throughout
    _, D = x_spread("bicgstab", op, y, e.k_clean)
    assert D < 1e-14


# ---------------- agreement window ----------------
def test_agreement_window_definition():
    h0 = np.array([1.0, 0.5, 0.25, 0.125, 0.0625])
    h1 = h0 * np.array([1, 1 + 1e-10, 1 + 1e-9, 1 + 5e-8, 1 + 1e-3])
    assert agreement_window([h0, h1], 1e-8) == 2
    assert agreement_window([h0, h1], 1e-7) == 3
    assert agreement_window([h0, h0], 1e-8) == 4
    h2 = h0 * np.array([1 + 2e-8, 1, 1, 1, 1])
    assert agreement_window([h0, h2], 1e-8) == -1
    assert agreement_window([h0, h1[:3]], 1e-8) == 2     # common length


def test_window_on_chaotic_proxy_and_noise_scaling():
    """Config 5 recipe at 24³ (rounding-chaotic BiCGSTAB): the member
    histories split before the end, the window ends exactly there, and a much
    larger noise ends it earlier (10⁶× here: the split is abrupt, 2e-14 and
    2e-16 both split at the same iteration on this problem)."""
    N = 24
    rp, ci, v = helmholtz_csr(N, kh=10 / 128)
    op, y = CsrOp(rp, ci, v), helmholtz_rhs(N)
    e = envelope("bicgstab", op, y, 1e-8, 2000)
    assert 0 < e.window < e.k_clean
    hists = [rel_history(oracle.solve("bicgstab", m, y, 1e-8, 2000))
             for m in [op] + [NoisyOp(op, s) for s in range(1, 9)]]
    L = min(map(len, hists))
    M = np.stack([h[:L] for h in hists])
    spread = (M.max(0) - M.min(0)) / M[0]
    np.testing.assert_array_equal(spread, e.hist_spread)
    # E3: the window is where the members agree to H/10 = 1e-9
    assert np.all(spread[:e.window + 1] <= 1e-9) and spread[e.window + 1] > 1e-9
    e_big = envelope("bicgstab", op, y, 1e-8, 2000, eps=2e-10, seeds=4)
    assert e_big.window < e.window
    # a history equal to the clean one passes, one off by 1e-6 inside the window fails
    assert e.history_error(e.hist_clean) == 0.0
    bad = e.hist_clean.copy()
    bad[e.window // 2] *= 1 + 1e-6
    assert e.history_error(bad) > e.H


# ---------------- FALSE_CONVERGENCE ----------------
def test_false_convergence_guard_boundary():
    """The guard's definition: > 10·tol flags, ≤ 10·tol does not.
    A = I, y = e₁, x̂ = (1 − δ)e₁ → true relative residual δ exactly."""
    g = json.load(open(GOLD))["guard_boundary"]
    n, delta = 4, 2.0 ** -20
    y = np.zeros(n, complex)
    y[0] = 1
    for ratio, want in ((g["ratio_converged"], CONVERGED), (g["ratio_false"], FALSE_CONVERGENCE)):
        op = _Ident(n, np.complex128)
        x = y * (1 - delta)
        res = Result(x=x, status=CONVERGED, iterations=3, matvecs_a=0, matvecs_ah=0, history=[1.0, delta])
        out = _finish(op, y, res, 1.0, delta / ratio, _Ctx(y))
        assert out.true_rel_res == delta
        assert out.status == want, (ratio, out.status_name)
    res = Result(x=y * (1 - delta), status=MAXIT, iterations=3, matvecs_a=0, matvecs_ah=0, history=[1.0])
    assert _finish(_Ident(n, complex), y, res, 1.0, delta / 100, _Ctx(y)).status == MAXIT   # only CONVERGED is re-labelled


def test_false_convergence_spec_fixture():
    """a seeded 8×8 system, CGS at tol 1e-15 near stagnation → the
    recurrence residual claims convergence, the true residual is > 10·tol."""
    g = json.load(open(GOLD))["spec_fixture"]
    A, y = graded_svd(n=8, decades=5, seed=5)
    r = oracle.solve(g["method"], DenseOp(A), y, g["tol"], g["maxit"])
    assert r.status_name == g["status"]
    assert r.rec_rel_res <= g["tol"]
    true = np.linalg.norm(y - A @ r.x) / np.linalg.norm(y)          # independent recomputation
    assert r.true_rel_res == pytest.approx(true, rel=1e-6)
    assert true > 10 * g["tol"]
    # the same system at a reachable tolerance converges for real
    r2 = oracle.solve(g["method"], DenseOp(A), y, 1e-9, g["maxit"])
    assert r2.status_name == "CONVERGED" and r2.true_rel_res <= 1e-8


@pytest.mark.parametrize("method", json.load(open(GOLD))["single_precision"]["methods"])
def test_false_convergence_single_precision(method):
    g = json.load(open(GOLD))["single_precision"]
    n = 256
    A = gauss_shifted_rows(n, 0, n, seed=1)
    y = cfg3_rhs(n)
    r = oracle.solve(method, DenseOp(A), y, g["tol"], g["maxit"])
    assert r.status_name == g["status"], (method, r.status_name)
    true = np.linalg.norm(y.astype(complex) - A.astype(complex) @ r.x.astype(complex)) / np.linalg.norm(y)
    assert true > 10 * g["tol"] and r.rec_rel_res <= g["tol"]


# ---------------- criterion (1) margin (reading E5) ----------------
def test_k_margin_tight_envelope_is_surveys_two():
    from oracle.envelope import k_margin
    assert k_margin(12, 12) == 2            # config 1: every member at 12
    assert k_margin(102, 110) == 2          # config 4 dense (102-110)
    assert k_margin(100, 109) == 3          # ⌈9/4⌉
    assert k_margin(1051, 1490) == 110      # config 5 BiCGSTAB, E = 32 (golden)


def test_k_margin_exceedance_rate():
    """The rule's purpose, measured independently of its formula: for E + 1 =
    33 members drawn from a normal distribution, an independent draw falls
    outside [k_min − m, k_max + m] with probability well under 1 % (the bare
    range: 2/(E+1) ≈ 6 %)."""
    from oracle.envelope import k_margin
    rng = np.random.default_rng(7)
    trials, out_bare, out_rule = 4000, 0, 0
    for _ in range(trials):
        ks = np.round(1260 + 120 * rng.standard_normal(33)).astype(int)
        new = int(round(1260 + 120 * rng.standard_normal()))
        lo, hi = int(ks.min()), int(ks.max())
        out_bare += not (lo <= new <= hi)
        m = k_margin(lo, hi)
        out_rule += not (lo - m <= new <= hi + m)
    assert 0.03 < out_bare / trials < 0.09
    assert out_rule / trials < 0.01


def test_check_k_uses_margin():
    e = oracle.envelope.Envelope(k_clean=1206, k_min=1051, k_max=1490, ks=[], statuses=[], window=22,
                                 hist_clean=np.ones(3))
    assert e.check_k(1024) and e.check_k(941) and not e.check_k(940)
    assert e.check_k(1600) and not e.check_k(1601)
    t = oracle.envelope.Envelope(k_clean=105, k_min=102, k_max=110, ks=[], statuses=[], window=5,
                                 hist_clean=np.ones(3))
    assert t.check_k(100) and not t.check_k(99) and t.check_k(112) and not t.check_k(113)
