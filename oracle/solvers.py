"""The five hot-path Krylov recurrences, step by step.  TEST INFRASTRUCTURE ONLY.

The paper names the methods and cites their sources but writes none of them
down (BiCGSTAB, CGNE, QMR: PIM90 set, §2.1, QMR "changed" per P:57 and
Chaumet's corrected version P:101 §6; BiCOR / CORS: Carpentieri, Jing & Huang
2011, §2.4).  The recurrences below follow SURVEY.md §8(c) O1-O5
line by line, in that notation, with the readings Q1-Q16 listed in
DESIGN.md §"Readings of the paper".  BiCG, CGS, CGNR and COCR (P:87
§3.4) — the SURVEY §8(f) NEXT-3 rows — follow the standard published
recurrences and double as pins of O4/O5: BiCOR ≡ BiCG(shadow Aᴴr₀*), CORS ≡
CGS(shadow Aᴴr₀*), BiCOR(r₀* = conj r₀) ≡ COCR on complex-symmetric A.

Common rules (SURVEY.md §8(c) "Common rules"):

* x₀ = 0 unless given; r₀ = y − A·x₀.
* stop when the recurrence residual satisfies ‖r_k‖² ≤ tol²·‖r₀‖²
  (equivalent to ‖r_k‖ ≤ tol·‖r₀‖; squared so that exact rational
  arithmetic needs no square root);
* ‖r₀‖ = 0 → CONVERGED with 0 iterations;
* a divisor that is exactly 0 → BREAKDOWN(name) (Q6), iterations =
  completed iterations; any non-finite scalar → NONFINITE;
* at exit the true residual ‖y − A·x̂‖/‖r₀‖ is recomputed;
  CONVERGED with true residual > 10·tol → FALSE_CONVERGENCE;
* ``iterations`` counts outer steps; ``matvecs_a/_ah`` count every
  operator application of the recurrence (setup included, the final
  true-residual check excluded).

Arithmetic is in the working precision of the inputs (complex64 or
complex128 numpy arrays), or exact (object arrays of
``exact.GaussianRational``), or mpmath (object arrays of ``mpmath.mpc``).
"""

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .numerics import dotc, dotu, norm_sq, sqrt

CONVERGED, MAXIT, BREAKDOWN, FALSE_CONVERGENCE, NONFINITE = 0, 1, 2, 3, 4
STATUS_NAMES = {0: "CONVERGED", 1: "MAXIT", 2: "BREAKDOWN",
                3: "FALSE_CONVERGENCE", 4: "NONFINITE"}
# breakdown codes (shared *numbering* with include/ccg.h; no code is shared)
BREAKDOWN_CODES = {None: 0, "rho": 1, "sigma": 2, "tt": 3, "omega": 4,
                   "pi": 5, "delta": 6, "epsilon": 7, "beta": 8, "xi": 9,
                   "vnorm": 10, "wnorm": 11, "gamma": 12}


@dataclass
class Result:
    x: np.ndarray
    status: int
    iterations: int
    matvecs_a: int
    matvecs_ah: int
    breakdown: Optional[str] = None
    rec_rel_res: float = float("nan")
    true_rel_res: float = float("nan")
    history: list = field(default_factory=list)   # ‖r_k‖ (recurrence), k = 0..
    half_step: bool = False                        # BiCGSTAB exit on ‖s‖

    @property
    def status_name(self):
        return STATUS_NAMES[self.status]


class _Breakdown(Exception):
    def __init__(self, name):
        super().__init__(name)
        self.name = name


class _NonFinite(Exception):
    pass


class _Ctx:
    """Per-solve scalar policy: keeps every scalar in the working precision."""

    def __init__(self, y, dots=None):
        self.obj = (y.dtype == object)
        # inner products (replaceable by a sharded implementation, oracle/sharded.py)
        self.dotc = dots.dotc if dots is not None else dotc
        self.dotu = dots.dotu if dots is not None else dotu
        self.norm_sq = dots.norm_sq if dots is not None else norm_sq
        if not self.obj:
            self.ctype = y.dtype.type                       # complex64/128
            self.rtype = np.finfo(y.dtype).dtype.type       # float32/64

    def c(self, s):
        return s if self.obj else self.ctype(s)

    def r(self, s):
        return s if self.obj else self.rtype(s)

    def check(self, *vals):
        if self.obj:
            return
        for v in vals:
            if not np.isfinite(v):
                raise _NonFinite()

    def div(self, num, den, name):
        if den == 0:
            raise _Breakdown(name)
        q = num / den
        self.check(q)
        return q


def _zero_like(y):
    if y.dtype == object:
        return np.array([0 * y[0]] * len(y), dtype=object) if len(y) else y.copy()
    return np.zeros_like(y)


def _init(op, y, x0):
    """x₀ and r₀ = y − A·x₀ (x₀ = 0 → r₀ = y with no matvec)."""
    if x0 is None:
        return _zero_like(y), y.copy()
    x = np.array(x0, dtype=y.dtype, copy=True)
    return x, y - op.apply(x)


def _finish(op, y, res, r0sq, tol, ctx):
    """True residual and FALSE_CONVERGENCE guard."""
    x = res.x
    rt = y - op.apply(x)
    if op is not None:                       # not counted as work
        op.n_a -= 1
    if ctx.obj:
        tr = float(ctx.norm_sq(rt)) ** 0.5
        r0 = float(r0sq) ** 0.5
    else:
        tr = float(np.sqrt(np.float64(ctx.norm_sq(rt.astype(np.complex128)))))
        r0 = float(np.sqrt(np.float64(r0sq)))
    res.true_rel_res = tr / r0 if r0 > 0 else 0.0
    if res.history:
        res.rec_rel_res = float(res.history[-1]) / r0 if r0 > 0 else 0.0
    if not ctx.obj and not np.all(np.isfinite(x)):
        res.status = NONFINITE
    if res.status == CONVERGED and res.true_rel_res > 10 * tol:
        res.status = FALSE_CONVERGENCE
    res.matvecs_a = op.n_a
    res.matvecs_ah = op.n_ah
    return res


def _run(body, op, y, tol, maxit, x0, dots=None, **kw):
    """Shared driver: setup, r0 check, exception → status mapping, finalize."""
    y = np.asarray(y)
    ctx = _Ctx(y, dots)
    op.reset_counts()
    x, r = _init(op, y, x0)
    r0sq = ctx.norm_sq(r)
    tol2 = tol * tol
    hist = [sqrt(r0sq)]
    state = {"x": x, "k": 0}
    res = Result(x=x, status=MAXIT, iterations=0, matvecs_a=0, matvecs_ah=0,
                 history=hist)
    if r0sq == 0:
        res.status = CONVERGED
        return _finish(op, y, res, r0sq, tol, ctx)
    try:
        status, k, half = body(op, y, x, r, r0sq, tol2, maxit, ctx, hist, state, **kw)
        res.status, res.iterations, res.half_step = status, k, half
    except _Breakdown as e:
        res.status, res.breakdown = BREAKDOWN, e.name
        res.iterations = state["k"] - 1
    except _NonFinite:
        res.status = NONFINITE
        res.iterations = state["k"] - 1
    res.x = state["x"]
    return _finish(op, y, res, r0sq, tol, ctx)


def _conv(rr, tol2, r0sq):
    return rr <= tol2 * r0sq


# ---------------------------------------------------------------------------
# O1 BiCGSTAB (van der Vorst).  Only A·x.  Shadow r̃ = r₀.
# ---------------------------------------------------------------------------
def _bicgstab(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st, shadow=None):
    rt = r.copy() if shadow is None else np.asarray(shadow, dtype=y.dtype)
    one = ctx.c(1)
    rho_prev = alpha = omega = one
    p = v = None
    for k in range(1, maxit + 1):
        st["k"] = k
        rho = ctx.c(ctx.dotc(rt, r))                               # ρ = ⟨r̃, r⟩
        ctx.check(rho)
        if rho == 0:
            raise _Breakdown("rho")
        if k == 1:
            p = r.copy()                                        # p = r
        else:
            beta = ctx.c((rho / rho_prev) * (alpha / omega))
            p = r + beta * (p - omega * v)                      # p = r + β(p − ωv)
        v = op.apply(p)                                         # v = A p
        sigma = ctx.c(ctx.dotc(rt, v))                              # σ = ⟨r̃, v⟩
        alpha = ctx.c(ctx.div(rho, sigma, "sigma"))             # α = ρ/σ
        s = r - alpha * v                                       # s = r − αv
        ss = ctx.r(ctx.norm_sq(s))
        ctx.check(ss)
        if _conv(ss, tol2, r0sq):                               # half-step exit (Q4)
            st["x"] = x = x + alpha * p
            hist.append(sqrt(ss))
            return CONVERGED, k, True
        t = op.apply(s)                                         # t = A s
        tt = ctx.r(ctx.norm_sq(t))
        ts = ctx.c(ctx.dotc(t, s))
        omega = ctx.c(ctx.div(ts, tt, "tt"))                    # ω = ⟨t,s⟩/⟨t,t⟩
        if omega == 0:
            raise _Breakdown("omega")
        st["x"] = x = x + alpha * p + omega * s                 # x += αp + ωs
        r = s - omega * t                                       # r = s − ωt
        rr = ctx.r(ctx.norm_sq(r))
        ctx.check(rr)
        hist.append(sqrt(rr))
        if _conv(rr, tol2, r0sq):
            return CONVERGED, k, False
        rho_prev = rho
    return MAXIT, maxit, False


# ---------------------------------------------------------------------------
# O2 CGNE (Craig's method = CG on AAᴴu = y, x = Aᴴu; Q1).
# ---------------------------------------------------------------------------
def _cgne(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st):
    p = op.apply_h(r)                                           # p = Aᴴ r
    rho = ctx.r(r0sq)                                           # ρ = ‖r‖²
    for k in range(1, maxit + 1):
        st["k"] = k
        pi = ctx.r(ctx.norm_sq(p))                                  # π = ‖p‖²
        alpha = ctx.r(ctx.div(rho, pi, "pi"))                   # α = ρ/π
        st["x"] = x = x + alpha * p                             # x += αp
        q = op.apply(p)
        r = r - alpha * q                                       # r −= α A p
        rho_new = ctx.r(ctx.norm_sq(r))
        ctx.check(rho_new)
        hist.append(sqrt(rho_new))
        if _conv(rho_new, tol2, r0sq):
            return CONVERGED, k, False
        if k == maxit:              # no further iterate needs the next direction
            break
        beta = ctx.r(rho_new / rho)
        p = op.apply_h(r) + beta * p                            # p = Aᴴr + βp
        rho = rho_new
    return MAXIT, maxit, False


# ---------------------------------------------------------------------------
# O3 QMR (Freund–Nachtigal without look-ahead, Templates form,
# M = I, Q2).  form="H": conjugated products and Aᴴ, w̃₁ = r₀.
# form="T": bilinear products and Aᵀ, w̃₁ = conj(r₀) (pin: identical iterates).
# ---------------------------------------------------------------------------
def _qmr(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st, form="H", shadow=None):
    if form == "H":
        ip, adj, cj = ctx.dotc, op.apply_h, (lambda z: z.conjugate())
        wt = r.copy() if shadow is None else np.asarray(shadow, dtype=y.dtype)
    else:
        ip, adj, cj = ctx.dotu, op.apply_t, (lambda z: z)
        wt = np.conj(r) if shadow is None else np.asarray(shadow, dtype=y.dtype)
    vt = r.copy()                                               # ṽ = r
    rho = ctx.r(sqrt(ctx.norm_sq(vt)))                              # ρ = ‖ṽ‖
    xi = ctx.r(sqrt(ctx.norm_sq(wt)))                               # ξ = ‖w̃‖
    gamma_prev = ctx.r(1)
    eta = ctx.c(-1)
    theta_prev = ctx.r(0)
    eps = None
    p = q = d = s = None
    for i in range(1, maxit + 1):
        st["k"] = i
        if rho == 0:
            raise _Breakdown("vnorm")
        if xi == 0:
            raise _Breakdown("wnorm")
        v = vt / rho                                            # v = ṽ/ρ
        w = wt / xi                                             # w = w̃/ξ
        delta = ctx.c(ip(w, v))                                 # δ = ⟨w, v⟩
        ctx.check(delta)
        if delta == 0:
            raise _Breakdown("delta")
        if i == 1:
            p = v.copy()
            q = w.copy()
        else:
            p = v - ctx.c(xi * delta / eps) * p                 # p = v − (ξδ/ε)p
            q = w - ctx.c(cj(rho * delta / eps)) * q            # q = w − conj(ρδ/ε)q
        pt = op.apply(p)                                        # p̃ = A p
        eps = ctx.c(ip(q, pt))                                  # ε = ⟨q, p̃⟩
        ctx.check(eps)
        if eps == 0:
            raise _Breakdown("epsilon")
        beta = ctx.c(eps / delta)                               # β = ε/δ
        if beta == 0:
            raise _Breakdown("beta")
        vt = pt - beta * v                                      # ṽ = p̃ − βv
        rho_next = ctx.r(sqrt(ctx.norm_sq(vt)))
        wt = adj(q) - ctx.c(cj(beta)) * w                       # w̃ = Aᴴq − conj(β)w
        xi_next = ctx.r(sqrt(ctx.norm_sq(wt)))
        theta = ctx.r(rho_next / (gamma_prev * abs(beta)))      # θ = ρ'/(γ_prev|β|)
        gamma = ctx.r(1 / sqrt(1 + theta * theta))              # γ = 1/√(1+θ²)
        ctx.check(theta, gamma)
        if gamma == 0:
            raise _Breakdown("gamma")
        eta = ctx.c(-eta * rho * gamma * gamma /
                    (beta * gamma_prev * gamma_prev))           # η
        if i == 1:
            d = eta * p
            s = eta * pt
        else:
            c2 = ctx.r((theta_prev * gamma) * (theta_prev * gamma))
            d = eta * p + c2 * d                                # d = ηp + (θ_prev γ)² d
            s = eta * pt + c2 * s                               # s = ηp̃ + (θ_prev γ)² s
        st["x"] = x = x + d                                     # x += d
        r = r - s                                               # r −= s
        rr = ctx.r(ctx.norm_sq(r))
        ctx.check(rr)
        hist.append(sqrt(rr))
        if _conv(rr, tol2, r0sq):
            return CONVERGED, i, False
        rho, xi, gamma_prev, theta_prev = rho_next, xi_next, gamma, theta
    return MAXIT, maxit, False


# ---------------------------------------------------------------------------
# O4 BiCOR (Carpentieri–Jing–Huang).  Shadow r₀* = r₀ (Q3).
# ---------------------------------------------------------------------------
def _bicor(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st, shadow=None):
    rs = r.copy() if shadow is None else np.array(shadow, dtype=y.dtype, copy=True)
    p = ps = q = None
    rho_prev = None
    for k in range(1, maxit + 1):
        st["k"] = k
        rh = op.apply(r)                                        # r̂ = A r
        rho = ctx.c(ctx.dotc(rs, rh))                               # ρ = ⟨r*, r̂⟩
        ctx.check(rho)
        if rho == 0:
            raise _Breakdown("rho")
        if k == 1:
            p, ps, q = r.copy(), rs.copy(), rh.copy()
        else:
            beta = ctx.c(rho / rho_prev)
            p = r + beta * p                                    # p = r + βp
            ps = rs + ctx.c(beta.conjugate()) * ps              # p* = r* + conj(β)p*
            q = rh + beta * q                                   # q = r̂ + βq
        qs = op.apply_h(ps)                                     # q* = Aᴴ p*
        xi = ctx.c(ctx.dotc(qs, q))                                 # ξ = ⟨q*, q⟩
        alpha = ctx.c(ctx.div(rho, xi, "xi"))                   # α = ρ/ξ
        st["x"] = x = x + alpha * p                             # x += αp
        r = r - alpha * q                                       # r −= αq
        rs = rs - ctx.c(alpha.conjugate()) * qs                 # r* −= conj(α)q*
        rr = ctx.r(ctx.norm_sq(r))
        ctx.check(rr)
        hist.append(sqrt(rr))
        if _conv(rr, tol2, r0sq):
            return CONVERGED, k, False
        rho_prev = rho
    return MAXIT, maxit, False


# ---------------------------------------------------------------------------
# O5 CORS.  BiCOR "squared"; transpose-free (Q15).  r₀* = r₀.
# ---------------------------------------------------------------------------
def _cors(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st, shadow=None):
    r0s = r.copy() if shadow is None else np.asarray(shadow, dtype=y.dtype)
    e = eh = qh = h = hh = None
    rho_prev = None
    for k in range(1, maxit + 1):
        st["k"] = k
        rh = op.apply(r)                                        # r̂ = A r
        rho = ctx.c(ctx.dotc(r0s, rh))                              # ρ = ⟨r₀*, r̂⟩
        ctx.check(rho)
        if rho == 0:
            raise _Breakdown("rho")
        if k == 1:
            e, eh, qh = r.copy(), rh.copy(), rh.copy()
        else:
            beta = ctx.c(rho / rho_prev)
            e = r + beta * h                                    # e = r + βh
            eh = rh + beta * hh                                 # ê = r̂ + βĥ
            qh = eh + beta * (hh + beta * qh)                   # q̂ = ê + β(ĥ + βq̂)
        q = op.apply(qh)                                        # q = A q̂
        xi = ctx.c(ctx.dotc(r0s, q))                                # ξ = ⟨r₀*, q⟩
        alpha = ctx.c(ctx.div(rho, xi, "xi"))                   # α = ρ/ξ
        h = e - alpha * qh                                      # h = e − αq̂
        hh = eh - alpha * q                                     # ĥ = ê − αq
        st["x"] = x = x + alpha * (e + h)                       # x += α(e + h)
        r = r - alpha * (eh + hh)                               # r −= α(ê + ĥ)
        rr = ctx.r(ctx.norm_sq(r))
        ctx.check(rr)
        hist.append(sqrt(rr))
        if _conv(rr, tol2, r0sq):
            return CONVERGED, k, False
        rho_prev = rho
    return MAXIT, maxit, False


# ---------------------------------------------------------------------------
# The rest of the catalogue on the same kernels:
# BiCG ("bigcg", §2.1), CGS (§2.1), CGNR ("cgmr" in P:57 §2.1, read
# as PIM's CGNR — DESIGN.md R5), COCR (§3.4, Sogabe–Zhang).  The paper
# writes none of them down; the recurrences are the standard published ones
# (BiCG/CGS/CGNR: Templates / PIM; COCR: Sogabe–Zhang 2007), in the same
# common rules as O1-O5.  They also serve as pins of O4/O5:
# BiCOR ≡ BiCG(shadow Aᴴr₀*), CORS ≡ CGS(shadow Aᴴr₀*), BiCOR(conj r₀) ≡ COCR.
# ---------------------------------------------------------------------------
def _bicg(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st, shadow=None):
    rt = r.copy() if shadow is None else np.array(shadow, dtype=y.dtype, copy=True)
    p = pt = None
    rho_prev = None
    for k in range(1, maxit + 1):
        st["k"] = k
        rho = ctx.c(ctx.dotc(rt, r))                            # ρ = ⟨r̃, r⟩
        ctx.check(rho)
        if rho == 0:
            raise _Breakdown("rho")
        if k == 1:
            p, pt = r.copy(), rt.copy()                         # p = r, p̃ = r̃
        else:
            beta = ctx.c(rho / rho_prev)                        # β = ρ/ρ_prev
            p = r + beta * p                                    # p = r + βp
            pt = rt + ctx.c(beta.conjugate()) * pt              # p̃ = r̃ + conj(β)p̃
        q = op.apply(p)                                         # q = A p
        qt = op.apply_h(pt)                                     # q̃ = Aᴴ p̃
        alpha = ctx.c(ctx.div(rho, ctx.c(ctx.dotc(pt, q)), "sigma"))   # α = ρ/⟨p̃, q⟩
        st["x"] = x = x + alpha * p                             # x += αp
        r = r - alpha * q                                       # r −= αq
        rt = rt - ctx.c(alpha.conjugate()) * qt                 # r̃ −= conj(α)q̃
        rr = ctx.r(ctx.norm_sq(r))
        ctx.check(rr)
        hist.append(sqrt(rr))
        if _conv(rr, tol2, r0sq):
            return CONVERGED, k, False
        rho_prev = rho
    return MAXIT, maxit, False


def _cgs(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st, shadow=None):
    rt = r.copy() if shadow is None else np.asarray(shadow, dtype=y.dtype)
    u = p = q = None
    rho_prev = None
    for k in range(1, maxit + 1):
        st["k"] = k
        rho = ctx.c(ctx.dotc(rt, r))                            # ρ = ⟨r̃, r⟩
        ctx.check(rho)
        if rho == 0:
            raise _Breakdown("rho")
        if k == 1:
            u = r.copy()                                        # u = r
            p = u.copy()                                        # p = u
        else:
            beta = ctx.c(rho / rho_prev)                        # β = ρ/ρ_prev
            u = r + beta * q                                    # u = r + βq
            p = u + beta * (q + beta * p)                       # p = u + β(q + βp)
        v = op.apply(p)                                         # v = A p
        alpha = ctx.c(ctx.div(rho, ctx.c(ctx.dotc(rt, v)), "sigma"))   # α = ρ/⟨r̃, v⟩
        q = u - alpha * v                                       # q = u − αv
        uq = u + q
        st["x"] = x = x + alpha * uq                            # x += α(u + q)
        r = r - alpha * op.apply(uq)                            # r −= α A(u + q)
        rr = ctx.r(ctx.norm_sq(r))
        ctx.check(rr)
        hist.append(sqrt(rr))
        if _conv(rr, tol2, r0sq):
            return CONVERGED, k, False
        rho_prev = rho
    return MAXIT, maxit, False


def _cocr(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st):
    """COCR (§3.4): for complex-symmetric A (A = Aᵀ) the CR recurrence
    with the unconjugated bilinear form [u, v] = Σ uᵢvᵢ; one A·x per iteration."""
    Ar = op.apply(r)                                            # A r₀
    p, Ap = r.copy(), Ar.copy()                                 # p = r, Ap = Ar
    mu = ctx.c(ctx.dotu(r, Ar))                                 # μ = [r, Ar]
    beta = None
    for k in range(1, maxit + 1):
        st["k"] = k
        if k > 1:
            p = r + beta * p                                    # p = r + βp
            Ap = Ar + beta * Ap                                 # Ap = Ar + βAp
        alpha = ctx.c(ctx.div(mu, ctx.c(ctx.dotu(Ap, Ap)), "xi"))   # α = μ/[Ap, Ap]
        st["x"] = x = x + alpha * p                             # x += αp
        r = r - alpha * Ap                                      # r −= αAp
        rr = ctx.r(ctx.norm_sq(r))
        ctx.check(rr)
        hist.append(sqrt(rr))
        if _conv(rr, tol2, r0sq):
            return CONVERGED, k, False
        if k == maxit:              # no further iterate needs A r (as CGNE, R2)
            break
        Ar = op.apply(r)                                        # A r
        mu_new = ctx.c(ctx.dotu(r, Ar))                         # μ' = [r, Ar]
        beta = ctx.c(ctx.div(mu_new, mu, "rho"))                # β = μ'/μ
        mu = mu_new
    return MAXIT, maxit, False


def _cgnr(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st):
    """CGNR (§2.1 "cgmr", read as PIM's CGNR — DESIGN.md R5): CG on the
    normal equations AᴴA x = Aᴴy; stops on the residual y − A·x of the original
    system like every other method (common rules)."""
    z = op.apply_h(r)                                           # z = Aᴴ r
    p = z.copy()                                                # p = z
    gamma = ctx.r(ctx.norm_sq(z))                               # γ = ‖z‖²
    for k in range(1, maxit + 1):
        st["k"] = k
        w = op.apply(p)                                         # w = A p
        alpha = ctx.r(ctx.div(gamma, ctx.r(ctx.norm_sq(w)), "pi"))     # α = γ/‖w‖²
        st["x"] = x = x + alpha * p                             # x += αp
        r = r - alpha * w                                       # r −= αw
        rr = ctx.r(ctx.norm_sq(r))
        ctx.check(rr)
        hist.append(sqrt(rr))
        if _conv(rr, tol2, r0sq):
            return CONVERGED, k, False
        if k == maxit:              # no further iterate needs the next direction
            break
        z = op.apply_h(r)                                       # z = Aᴴ r
        gamma_new = ctx.r(ctx.norm_sq(z))
        beta = ctx.r(gamma_new / gamma)                         # β = γ'/γ
        p = z + beta * p                                        # p = z + βp
        gamma = gamma_new
    return MAXIT, maxit, False


def _tfqmr(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st, shadow=None):
    """TFQMR (§2.1: "QMR and TFQMR algorithms are in this version
    changed"; Freund's transpose-free QMR, Saad Alg. 7.8 restated in pairs of
    half-steps m = 2k−2, 2k−1).  TFQMR carries no residual vector: the stopping
    test is Freund's bound ‖r_m‖ ≤ τ_m·√(m+1) ≤ tol·‖r₀‖ (R9); an exit
    after the first half of pair k reports iteration k with half_step (R10);
    shadow r₀* = r₀ (R11)."""
    st["k"] = 1                     # the setup product and α belong to iteration 1
    rs = r.copy() if shadow is None else np.asarray(shadow, dtype=y.dtype)
    w = r.copy()                                                # w₀ = r₀
    u = r.copy()                                                # u₀ = r₀
    v = op.apply(u)                                             # v₀ = A u₀
    d = _zero_like(y)                                           # d₀ = 0
    tau = ctx.r(sqrt(r0sq))                                     # τ₀ = ‖r₀‖
    theta = ctx.r(0)
    eta = ctx.c(0)
    rho = ctx.c(ctx.dotc(rs, r))                                # ρ₀ = ⟨r₀*, r₀⟩
    ctx.check(rho)
    if rho == 0:
        raise _Breakdown("rho")
    alpha = ctx.c(ctx.div(rho, ctx.c(ctx.dotc(rs, v)), "sigma"))    # α = ρ/⟨r₀*, v⟩
    au_even = v                                                 # A u₀ = v₀ (u₀ = p₀ = r₀)
    u2 = au = None
    bound2 = r0sq
    for k in range(1, maxit + 1):
        st["k"] = k
        for half in (0, 1):
            if half == 0:
                u2 = u - alpha * v                              # u_{m+1} = u_m − α v_m
                au, um = au_even, u                             # A u_m, kept from the last product (m even)
            else:
                au, um = op.apply(u2), u2                       # A u_m        (m odd)
            w = w - alpha * au                                  # w_{m+1} = w_m − α A u_m
            d = um + ctx.c(theta * theta * eta / alpha) * d     # d_{m+1} = u_m + (θ_m² η_m/α) d_m
            theta = ctx.r(sqrt(ctx.norm_sq(w)) / tau)           # θ_{m+1} = ‖w_{m+1}‖/τ_m
            cc = ctx.r(1 / sqrt(1 + theta * theta))             # c_{m+1} = 1/√(1+θ²)
            tau = ctx.r(tau * theta * cc)                       # τ_{m+1} = τ_m θ c
            eta = ctx.c(cc * cc * alpha)                        # η_{m+1} = c² α
            ctx.check(theta, tau, eta)
            st["x"] = x = x + eta * d                           # x_{m+1} = x_m + η d
            bound2 = ctx.r(tau * tau * (2 * k + half))          # (τ_{m+1}·√(m+2))²
            if _conv(bound2, tol2, r0sq):
                hist.append(sqrt(bound2))
                return CONVERGED, k, half == 0
        hist.append(sqrt(bound2))
        if k == maxit:              # no further iterate needs the next products (R2)
            break
        rho_new = ctx.c(ctx.dotc(rs, w))                        # ρ_{m+1} = ⟨r₀*, w_{m+1}⟩
        ctx.check(rho_new)
        if rho_new == 0:
            raise _Breakdown("rho")
        beta = ctx.c(rho_new / rho)                             # β = ρ_{m+1}/ρ_{m−1}
        rho = rho_new
        u = w + beta * u2                                       # u_{m+1} = w + β u_m
        au_even = op.apply(u)                                   # A u_{m+1}
        v = au_even + beta * (au + beta * v)                    # v = A u + β(A u_m + β v)
        alpha = ctx.c(ctx.div(rho, ctx.c(ctx.dotc(rs, v)), "sigma"))
    return MAXIT, maxit, False


def _gmres(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st, restart=30):
    """Restarted GMRES(m) ("rgmres", §2.1): Arnoldi
    with classical Gram–Schmidt applied twice (CGS2, R13), complex
    Givens rotations, back substitution at the end of a cycle; the stopping
    test is the Givens residual |g_{j+1}| ≤ tol·‖r₀‖ (the recurrence residual,
    R15); a restart recomputes r = y − A·x explicitly (one product, R14);
    ``iterations`` counts Arnoldi steps (one A·x each)."""
    m = int(restart)
    k = 0
    rr = r0sq
    while True:
        beta = ctx.r(sqrt(rr))
        V = [r / beta]                                          # v₁ = r/β
        R = []                                                  # rotated columns of H
        cs, sn = [], []
        g = [ctx.c(beta)]                                       # g = β e₁
        for j in range(m):
            k += 1
            st["k"] = k
            w = op.apply(V[j])                                  # w = A v_j
            h = [ctx.c(ctx.dotc(V[i], w)) for i in range(j + 1)]      # h = Vᴴw
            for i in range(j + 1):
                w = w - h[i] * V[i]                             # w −= V h
            h2 = [ctx.c(ctx.dotc(V[i], w)) for i in range(j + 1)]     # second pass (CGS2)
            for i in range(j + 1):
                w = w - h2[i] * V[i]
            h = [ctx.c(a + b) for a, b in zip(h, h2)]
            hn = ctx.r(sqrt(ctx.norm_sq(w)))                    # h_{j+1,j} = ‖w‖
            ctx.check(hn, *h)
            for i in range(j):                                  # previous rotations
                a, b = h[i], h[i + 1]
                h[i] = ctx.c(cs[i] * a + sn[i] * b)
                h[i + 1] = ctx.c(-sn[i].conjugate() * a + cs[i] * b)
            a = h[j]                                            # new rotation zeroing h_{j+1,j}
            if a == 0:
                c, s_ = ctx.r(0), ctx.c(1)
            else:
                aa = abs(a)
                nu = ctx.r(sqrt(aa * aa + hn * hn))
                c, s_ = ctx.r(aa / nu), ctx.c((a / aa) * (hn / nu))
            cs.append(c)
            sn.append(s_)
            h[j] = ctx.c(c * a + s_ * hn)
            g.append(ctx.c(-s_.conjugate() * g[j]))             # g_{j+1} = −conj(s) g_j
            g[j] = ctx.c(c * g[j])                              # g_j = c g_j
            R.append(h)
            res = abs(g[j + 1])
            hist.append(res)
            conv = _conv(res * res, tol2, r0sq)
            if conv or k == maxit or j == m - 1:
                yv = [None] * (j + 1)                           # back substitution R y = g
                for i in range(j, -1, -1):
                    t = g[i]
                    for l in range(i + 1, j + 1):
                        t = t - R[l][i] * yv[l]
                    yv[i] = ctx.c(ctx.div(t, R[i][i], "gamma"))
                for i in range(j + 1):
                    x = x + yv[i] * V[i]                        # x += V y
                st["x"] = x
                if conv:
                    return CONVERGED, k, False
                if k == maxit:
                    return MAXIT, k, False
                break
            V.append(w / hn)                                    # v_{j+1} = w/h_{j+1,j}
        r = y - op.apply(x)                                     # restart: explicit residual
        rr = ctx.r(ctx.norm_sq(r))
        ctx.check(rr)
        if _conv(rr, tol2, r0sq):
            return CONVERGED, k, False


def _small_solve(Z, z, ctx, name):
    """Gaussian elimination with partial pivoting on a small ℓ×ℓ system (any
    scalar type: working precision, exact rationals, mpmath)."""
    n = len(z)
    M = [list(row) + [zi] for row, zi in zip(Z, z)]
    for c in range(n):
        p = max(range(c, n), key=lambda i: M[i][c].real * M[i][c].real + M[i][c].imag * M[i][c].imag)
        if M[p][c] == 0:
            raise _Breakdown(name)
        M[c], M[p] = M[p], M[c]
        for i in range(c + 1, n):
            f = M[i][c] / M[c][c]
            for j in range(c, n + 1):
                M[i][j] = M[i][j] - f * M[c][j]
    g = [None] * n
    for i in range(n - 1, -1, -1):
        t = M[i][n]
        for j in range(i + 1, n):
            t = t - M[i][j] * g[j]
        g[i] = ctx.c(t / M[i][i])
    return g


def _bicgstabl(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st, ell=2, shadow=None, trace=None):
    """BiCGstab(ℓ) (§3.1, the "vanilla" algorithm of Sleijpen–Fokkema;
    SURVEY §8(f) NEXT-3): per cycle ℓ BiCG steps (two A·x each) build r̂₀..r̂_ℓ,
    û₀..û_ℓ with r̂_{j+1} = A r̂_j; the minimal-residual part then minimises
    ‖r̂₀ − Σ_{j=1..ℓ} γ_j r̂_j‖ through the normal equations Z γ = z,
    Z_ij = ⟨r̂_i, r̂_j⟩, z_i = ⟨r̂_i, r̂₀⟩ (R16-R18).  ``iterations``
    counts BiCG steps; r̂₀ is the current residual after every step, so the
    stopping test runs after every step and after the MR part.  ℓ = 1 is
    BiCGSTAB (pinned)."""
    L = int(ell)
    rt = r.copy() if shadow is None else np.asarray(shadow, dtype=y.dtype)
    R = [r.copy()] + [None] * L
    U = [_zero_like(y)] + [None] * L
    rho0, alpha, omega = ctx.c(1), ctx.c(0), ctx.c(1)
    k = 0
    while True:
        rho0 = ctx.c(-omega * rho0)                                 # ρ₀ = −ω ρ₀
        for j in range(L):                                          # BiCG part
            k += 1
            st["k"] = k
            rho1 = ctx.c(ctx.dotc(rt, R[j]))                        # ρ₁ = ⟨r̃, r̂_j⟩
            ctx.check(rho1)
            beta = ctx.c(alpha * ctx.div(rho1, rho0, "rho"))        # β = α ρ₁/ρ₀
            rho0 = rho1
            for i in range(j + 1):
                U[i] = R[i] - beta * U[i]                           # û_i = r̂_i − β û_i
            U[j + 1] = op.apply(U[j])                               # û_{j+1} = A û_j
            gam = ctx.c(ctx.dotc(rt, U[j + 1]))                     # γ = ⟨r̃, û_{j+1}⟩
            alpha = ctx.c(ctx.div(rho0, gam, "sigma"))              # α = ρ₀/γ
            for i in range(j + 1):
                R[i] = R[i] - alpha * U[i + 1]                      # r̂_i −= α û_{i+1}
            st["x"] = x = x + alpha * U[0]                          # x += α û₀
            rr = ctx.r(ctx.norm_sq(R[0]))                           # r̂₀ is the residual of x
            ctx.check(rr)
            hist.append(sqrt(rr))
            if _conv(rr, tol2, r0sq):
                return CONVERGED, k, False
            if k == maxit and j < L - 1:                            # mid-cycle: no MR part
                return MAXIT, k, False
            R[j + 1] = op.apply(R[j])                               # r̂_{j+1} = A r̂_j
        # MR part: Z γ = z
        Z = [[ctx.c(ctx.dotc(R[i], R[jj])) for jj in range(1, L + 1)] for i in range(1, L + 1)]
        zv = [ctx.c(ctx.dotc(R[i], R[0])) for i in range(1, L + 1)]
        g = _small_solve(Z, zv, ctx, "omega")
        omega = g[L - 1]                                            # ω = γ_ℓ
        for jj in range(1, L + 1):
            x = x + g[jj - 1] * R[jj - 1]                           # x += Σ γ_j r̂_{j−1}
        st["x"] = x
        for jj in range(1, L + 1):
            R[0] = R[0] - g[jj - 1] * R[jj]                         # r̂₀ −= Σ γ_j r̂_j
        for jj in range(1, L + 1):
            U[0] = U[0] - g[jj - 1] * U[jj]                         # û₀ −= Σ γ_j û_j
        if trace is not None:                                       # pins only
            trace(R, U)
        rr = ctx.r(ctx.norm_sq(R[0]))
        ctx.check(rr)
        hist[-1] = sqrt(rr)                                         # the residual of iteration k
        if _conv(rr, tol2, r0sq):
            return CONVERGED, k, False
        if k >= maxit:
            return MAXIT, k, False
        if omega == 0:
            raise _Breakdown("omega")


def _pbicgstab(op, y, x, r, r0sq, tol2, maxit, ctx, hist, st, shadow=None):
    """Pipelined BiCGSTAB (SURVEY §8(f) NEXT-2 iii; Cools–Vanroose's
    communication-hiding form): the same iterates as O1 in exact arithmetic
    (pinned), with the auxiliary recurrences s = A p, z = A s, w = A r,
    t = A w, v = A z so that each iteration needs TWO reduction phases, each
    independent of the product that follows it ({⟨q,y⟩, ⟨y,y⟩, ‖q‖²} ∥ v = A z;
    {⟨r̃,r⟩, ⟨r̃,w⟩, ⟨r̃,s⟩, ⟨r̃,z⟩, ‖r‖²} ∥ t = A w).  Half-step exit on ‖q‖ (q is
    O1's s) as Q4."""
    rt = r.copy() if shadow is None else np.asarray(shadow, dtype=y.dtype)
    st["k"] = 1                         # the setup products and α₀ belong to iteration 1
    w = op.apply(r)                                             # w₀ = A r₀
    t = op.apply(w)                                             # t₀ = A w₀
    rho = ctx.c(ctx.dotc(rt, r))                                # ρ₀ = ⟨r̃, r₀⟩
    ctx.check(rho)
    if rho == 0:
        raise _Breakdown("rho")
    alpha = ctx.c(ctx.div(rho, ctx.c(ctx.dotc(rt, w)), "sigma"))   # α₀ = ρ₀/⟨r̃, w₀⟩
    beta = omega = ctx.c(0)
    p = s = z = v = None
    for k in range(1, maxit + 1):
        st["k"] = k
        if k == 1:
            p, s, z = r.copy(), w.copy(), t.copy()
        else:
            p = r + beta * (p - omega * s)                      # p = r + β(p − ωs)
            s = w + beta * (s - omega * z)                      # s = w + β(s − ωz)
            z = t + beta * (z - omega * v)                      # z = t + β(z − ωv)
        q = r - alpha * s                                       # q = r − αs
        yv = w - alpha * z                                      # y = w − αz
        qq = ctx.r(ctx.norm_sq(q))
        ctx.check(qq)
        if _conv(qq, tol2, r0sq):                               # half-step exit (Q4)
            st["x"] = x = x + alpha * p
            hist.append(sqrt(qq))
            return CONVERGED, k, True
        qy = ctx.c(ctx.dotc(yv, q))                             # ⟨y, q⟩
        yy = ctx.r(ctx.norm_sq(yv))                             # ⟨y, y⟩
        v = op.apply(z)                                         # v = A z
        omega = ctx.c(ctx.div(qy, yy, "tt"))                    # ω = ⟨y,q⟩/⟨y,y⟩
        if omega == 0:
            raise _Breakdown("omega")
        st["x"] = x = x + alpha * p + omega * q                 # x += αp + ωq
        r = q - omega * yv                                      # r = q − ωy
        w = yv - omega * (t - alpha * v)                        # w = y − ω(t − αv)
        rr = ctx.r(ctx.norm_sq(r))
        ctx.check(rr)
        hist.append(sqrt(rr))
        if _conv(rr, tol2, r0sq):
            return CONVERGED, k, False
        if k == maxit:              # no further iterate needs the next products (R2)
            break
        rho_new = ctx.c(ctx.dotc(rt, r))                        # ⟨r̃, r⟩
        rw = ctx.c(ctx.dotc(rt, w))                             # ⟨r̃, w⟩
        rs_ = ctx.c(ctx.dotc(rt, s))                            # ⟨r̃, s⟩
        rz = ctx.c(ctx.dotc(rt, z))                             # ⟨r̃, z⟩
        t = op.apply(w)                                         # t = A w
        ctx.check(rho_new)
        if rho_new == 0:
            raise _Breakdown("rho")
        beta = ctx.c((alpha / omega) * (rho_new / rho))         # β = (α/ω) ρ'/ρ
        rho = rho_new
        alpha = ctx.c(ctx.div(rho, ctx.c(rw + beta * rs_ - beta * omega * rz), "sigma"))
    return MAXIT, maxit, False


METHODS = {
    "bicgstab": _bicgstab, "cgne": _cgne, "qmr": _qmr, "bicor": _bicor,
    "cors": _cors,
    # SURVEY §8(f) NEXT-3
    "bicg": _bicg, "cgs": _cgs, "cocr": _cocr, "cgnr": _cgnr, "tfqmr": _tfqmr,
    "gmres": _gmres, "bicgstabl": _bicgstabl,
    "pbicgstab": _pbicgstab,    # NEXT-2 (iii)
}
HOT_PATH = ("bicgstab", "cgne", "qmr", "bicor", "cors")
NEXT3 = ("bicg", "cgs", "cocr", "cgnr", "tfqmr", "gmres", "bicgstabl")
NEXT2 = ("pbicgstab",)


def solve(method, op, y, tol, maxit, x0=None, dots=None, **kw):
    """Run ``method`` on A x = y (A given as an operator with apply/apply_h/apply_t).

    Returns a :class:`Result`.  ``kw`` passes method options (``shadow`` for
    BiCGSTAB/BiCOR/CORS/BiCG/CGS/QMR, ``form`` for QMR)."""
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}")
    return _run(METHODS[method], op, y, tol, maxit, x0, dots=dots, **kw)


def solve_jacobi(method, op, d, y, tol, maxit, x0=None, **kw):
    """Right-Jacobi-preconditioned solve: run ``method``
    on B u = y with B = A·diag(d)⁻¹ (u₀ = D x₀), return x = D⁻¹u in the Result
    (true residual recomputed by the wrapper, i.e. y − A x)."""
    from .operators import JacobiRightOp
    B = JacobiRightOp(op, d)
    u0 = None if x0 is None else np.asarray(d) * np.asarray(x0)
    res = solve(method, B, y, tol, maxit, x0=u0, **kw)
    res.x = (B.dinv * res.x).astype(res.x.dtype)
    return res
