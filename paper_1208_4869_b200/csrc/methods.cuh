// methods.cuh — the five recurrences of the hot path, split into phases.
//
// Each phase is (a) a per-element functor run inside a matvec epilogue or a
// fused vector pass, accumulating up to K fp64 partial sums, and (b) a
// single-thread `finish` that turns the sums into the recurrence scalars,
// applies the stopping / breakdown rules and updates the device State.
//
// Recurrences: BiCGSTAB, CGNE, QMR — PIM90 set, PAPER.md P:57 [§2.1] (QMR as
// corrected, P:101 [§6]); BiCOR, CORS — P:69 [§2.4].  The paper writes none
// of them down; the formulation followed is SURVEY.md §8(c) O1-O5 (restated
// in DESIGN.md), with the paper readings Q1-Q16.  Stopping rule
// ‖r_k‖² ≤ tol²‖r_0‖², breakdown = a divisor exactly 0 (Q6),
// NaN/Inf scalar => NONFINITE.
//
// Vector updates run in the working precision T; scalars are fp64 and are
// rounded to T once per kernel (load()).
#pragma once
#include "common.cuh"

namespace ccg {

template <typename T> using Cx = typename CT<T>::c;

__device__ __forceinline__ void conv_check_common(State* st, int k, double rr, bool& stop) {
  // rr non-finite -> NONFINITE with k-1 completed; converged -> k; maxit -> k
  stop = true;
  if (!isfinite(rr)) { set_done(st, ST_NONFINITE, k - 1); return; }
  push_hist(st, k, rr);
  if (rr <= st->tol2r0) { set_done(st, ST_CONVERGED, k); return; }
  if (k >= st->maxit) { set_done(st, ST_MAXIT, k); return; }
  stop = false;
}

// ===========================================================================
// Generic phases
// ===========================================================================
// r = y (pass) or r = y − A·x0 (gemv epilogue); copies r into up to three
// more vectors (shadow residuals etc.); K=1: ‖r‖².
template <typename T>
struct InitR {
  static constexpr int K = 1;
  using C = Cx<T>;
  const C* y;
  C *d0, *d1, *d2, *d3;
  __device__ void load(const State*) {}
  __device__ void put(int64_t i, C r, double2* acc) {
    if (d0) d0[i] = r;
    if (d1) d1[i] = r;
    if (d2) d2[i] = r;
    if (d3) d3[i] = r;
    nrm_acc(acc[0], r);
  }
  __device__ void operator()(int64_t i, double2* acc) { put(i, y[i], acc); }        // pass
  __device__ void operator()(int64_t i, C ax, double2* acc) { put(i, csub(y[i], ax), acc); }  // epilogue
  static __device__ void finish(State* st, const double2* s) {
    const double rr = s[0].x;
    st->r0sq = rr;
    st->tol2r0 = st->tol2 * rr;
    st->rr = rr;
    if (st->hist && st->hist_cap > 0) st->hist[0] = rr > 0 ? 1.0 : 0.0;
    if (!isfinite(rr)) { set_done(st, ST_NONFINITE, 0); return; }
    if (rr == 0.0) { set_done(st, ST_CONVERGED, 0); return; }
    switch (st->method) {
      case M_BICGSTAB:
      case M_BICG:
      case M_PBICGSTAB:
      case M_CGS: st->rho = make_double2(rr, 0.0); break;
      case M_GMRES: {
        GmDev* gm = reinterpret_cast<GmDev*>(st->gm);
        gm->g[0] = make_double2(sqrt(rr), 0.0);
        gm->j = 0; gm->k = 0; gm->pend = -1;
        gm->endflag = 0; gm->noend = 1; gm->noxupd = 1; gm->norestart = 1;
        break;
      }
      case M_BICGSTABL:
        // ρ₀ = −ω·1 = −1 at the first cycle start; step 1: ρ₁ = ⟨r̃, r₀⟩ = ‖r₀‖²,
        // β = α·(ρ₁/ρ₀) with α = 0, ρ₀ ← ρ₁
        st->alpha = make_double2(0.0, 0.0);
        st->omega = make_double2(1.0, 0.0);
        st->beta = zmul(st->alpha, zdiv(make_double2(rr, 0.0), make_double2(-1.0, 0.0)));
        st->rho = make_double2(rr, 0.0);
        break;
      case M_TFQMR:
        st->rho = make_double2(rr, 0.0);
        st->tau = sqrt(rr); st->theta = 0.0; st->eta = make_double2(0.0, 0.0);
        break;
      case M_CGNE: st->rho_r = rr; break;
      case M_QMR:
        st->rnrm = sqrt(rr); st->xnrm = sqrt(rr);
        st->gamma_prev = 1.0; st->eta = make_double2(-1.0, 0.0); st->theta_prev = 0.0;
        break;
      default: break;
    }
  }
};

// out[i] = value (ccg_apply, multi-GPU Aᴴ full-length result)
template <typename T>
struct Store {
  static constexpr int K = 0;
  using C = Cx<T>;
  C* out;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C v, double2*) { out[i] = v; }
  static __device__ void finish(State*, const double2*) {}
};

// dst[i] = src[i]
template <typename T>
struct Copy {
  static constexpr int K = 0;
  using C = Cx<T>;
  const C* src;
  C* dst;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, double2*) { dst[i] = src[i]; }
  static __device__ void finish(State*, const double2*) {}
};

// ‖y − A·x‖² at exit
template <typename T>
struct TrueRes {
  static constexpr int K = 1;
  using C = Cx<T>;
  const C* y;
  __device__ void load(const State*) {}
  using Pre = C;   // early load (matvec.cuh EpiPre)
  __device__ Pre pre(int64_t i) const { return y[i]; }
  __device__ void post(int64_t, C ax, Pre yi, double2* acc) { nrm_acc(acc[0], csub(yi, ax)); }
  __device__ void operator()(int64_t i, C ax, double2* acc) { post(i, ax, pre(i), acc); }
  static __device__ void finish(State* st, const double2* s) { st->true_rr = s[0].x; }
};

// ===========================================================================
// O1 BiCGSTAB.  Per iteration: P → [A p → v, σ] → S → [A s → t, ⟨t,s⟩,⟨t,t⟩] → X
// ===========================================================================
// the direction update p = r (k=1) | r + β(p − ωv): one definition shared by
// the pass (BsP) and the fused form (BsPIn / BsV2), so both give the same bits
template <typename C>
__device__ __forceinline__ C bs_pnew(C r, C p, C v, C beta, C omega, int first) {
  return first ? r : caxpy(r, beta, caxmy(p, omega, v));
}

template <typename T>
struct BsP {  // p = r (k=1) | p = r + β(p − ωv)
  static constexpr int K = 0;
  using C = Cx<T>;
  const C* r; C* p; const C* v;
  C beta, omega; int first;
  __device__ void load(const State* st) {
    first = st->iter == 0;
    beta = fromd2<C>(st->beta); omega = fromd2<C>(st->omega);
  }
  __device__ void operator()(int64_t i, double2*) { p[i] = bs_pnew(r[i], p[i], v[i], beta, omega, first); }
  static __device__ void finish(State*, const double2*) {}
};

template <typename T>
struct BsV {  // v = A p ; σ = ⟨r̃, v⟩ ; α = ρ/σ
  static constexpr int K = 1;
  using C = Cx<T>;
  C* v; const C* rt;
  __device__ void load(const State*) {}
  // early load of the epilogue input (issued with the product's loads; matvec.cuh EpiPre)
  using Pre = C;
  __device__ Pre pre(int64_t i) const { return rt[i]; }
  __device__ void post(int64_t i, C val, Pre b, double2* acc) { v[i] = val; dotc_acc(acc[0], b, val); }
  __device__ void operator()(int64_t i, C val, double2* acc) { post(i, val, pre(i), acc); }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter + 1;
    st->matvecs_a++;
    const double2 sigma = s[0];
    if (zzero(sigma)) { set_done(st, ST_BREAKDOWN, k - 1, BD_SIGMA); return; }
    st->alpha = zdiv(st->rho, sigma);
    if (!zfinite(st->alpha)) { set_done(st, ST_NONFINITE, k - 1); return; }
  }
};

template <typename T>
struct BsS {  // s = r − αv ; ‖s‖² ; half-step test (Q4)
  static constexpr int K = 1;
  using C = Cx<T>;
  const C* r; const C* v; C* s;
  C alpha;
  __device__ void load(const State* st) { alpha = fromd2<C>(st->alpha); }
  __device__ void operator()(int64_t i, double2* acc) {
    const C si = caxmy(r[i], alpha, v[i]);
    s[i] = si;
    nrm_acc(acc[0], si);
  }
  static __device__ void finish(State* st, const double2* sm) {
    const int k = st->iter + 1;
    const double ss = sm[0].x;
    if (!isfinite(ss)) { set_done(st, ST_NONFINITE, k - 1); return; }
    st->ss = ss;
    if (ss <= st->tol2r0) { st->half = 1; st->gate2 = 1; }
  }
};

template <typename T>
struct BsT {  // t = A s ; ⟨t,s⟩, ⟨t,t⟩ ; ω
  static constexpr int K = 2;
  using C = Cx<T>;
  C* t; const C* s;
  __device__ void load(const State*) {}
  using Pre = C;   // early load (matvec.cuh EpiPre)
  __device__ Pre pre(int64_t i) const { return s[i]; }
  __host__ __device__ const void* pre_src() const { return s; }   // the product's own input: no second load (EpiPreSrc)
  __device__ void post(int64_t i, C val, Pre si, double2* acc) {
    t[i] = val;
    dotc_acc(acc[0], val, si);
    nrm_acc(acc[1], val);
  }
  __device__ void operator()(int64_t i, C val, double2* acc) { post(i, val, pre(i), acc); }
  static __device__ void finish(State* st, const double2* sm) {
    const int k = st->iter + 1;
    st->matvecs_a++;
    const double tt = sm[1].x;
    if (tt == 0.0) { set_done(st, ST_BREAKDOWN, k - 1, BD_TT); return; }
    st->omega = make_double2(sm[0].x / tt, sm[0].y / tt);
    if (!zfinite(st->omega)) { set_done(st, ST_NONFINITE, k - 1); return; }
    if (zzero(st->omega)) { set_done(st, ST_BREAKDOWN, k - 1, BD_OMEGA); return; }
  }
};

// ---- BiCGSTAB with the P and S passes folded into the products (single GPU,
// dense split GEMV with several strips; Engine::matvec_a_in; the S fold alone
// also on the stencil and the SELL SpMV, Engine::in_fuse_ro_ok).  The GEMV forms
// each staged x element with BsPIn / BsSIn while it loads the strip, and the
// strip-sum epilogue (after every CTA has read the old vectors) recomputes the
// same element for its own row and stores it: 5 launches per iteration
// instead of 7, same recurrence values bit for bit except ‖s‖², whose partial
// sums now run in the epilogue's grid order (it only feeds the half-step test).
template <typename T>
struct BsPIn {   // staged element of p = r + β(p − ωv)
  using C = Cx<T>;
  const C* r; const C* p; const C* v;
  C beta, omega; int first;
  __device__ void load(const State* st) {
    first = st->iter == 0;
    beta = fromd2<C>(st->beta); omega = fromd2<C>(st->omega);
  }
  __device__ C operator()(const C*, int64_t j) const { return bs_pnew(r[j], p[j], v[j], beta, omega, first); }
};

template <typename T>
struct BsV2 {   // p_i stored, v = A p, σ = ⟨r̃, v⟩
  static constexpr int K = 1;
  using C = Cx<T>;
  C* v; const C* rt; const C* r; C* p;
  C beta, omega; int first;
  __device__ void load(const State* st) {
    first = st->iter == 0;
    beta = fromd2<C>(st->beta); omega = fromd2<C>(st->omega);
  }
  __device__ void operator()(int64_t i, C val, double2* acc) {
    p[i] = bs_pnew(r[i], p[i], v[i], beta, omega, first);
    const C b = rt[i];
    v[i] = val;
    dotc_acc(acc[0], b, val);
  }
  static __device__ void finish(State* st, const double2* s) { BsV<T>::finish(st, s); }
};

template <typename T>
struct BsSIn {   // staged element of s = r − αv
  using C = Cx<T>;
  const C* r; const C* v;
  C alpha;
  __device__ void load(const State* st) { alpha = fromd2<C>(st->alpha); }
  // r and v are read-only for the whole product (the non-coherent path)
  __device__ C operator()(const C*, int64_t j) const { return caxmy(__ldg(r + j), alpha, __ldg(v + j)); }
};

template <typename T>
struct BsT2 {   // s_i stored, t = A s ; ⟨t,s⟩, ⟨t,t⟩, ‖s‖² ; half-step test, then ω
  static constexpr int K = 3;
  using C = Cx<T>;
  C* t; C* s; const C* r; const C* v;
  C alpha;
  __device__ void load(const State* st) { alpha = fromd2<C>(st->alpha); }
  __device__ void operator()(int64_t i, C val, double2* acc) {
    const C si = caxmy(r[i], alpha, v[i]);
    s[i] = si;
    t[i] = val;
    dotc_acc(acc[0], val, si);
    nrm_acc(acc[1], val);
    nrm_acc(acc[2], si);
  }
  static __device__ void finish(State* st, const double2* sm) {
    const int k = st->iter + 1;
    const double ss = sm[2].x;
    if (!isfinite(ss)) { set_done(st, ST_NONFINITE, k - 1); return; }
    st->ss = ss;
    // half-step exit (Q4): t = A s was formed but is not part of the method
    // (not counted; BsX does x += αp)
    if (ss <= st->tol2r0) { st->half = 1; st->gate2 = 1; return; }
    BsT<T>::finish(st, sm);
  }
};

template <typename T>
struct BsX {  // x += αp + ωs ; r = s − ωt ; ‖r‖², ⟨r̃, r⟩   (half-step: x += αp)
  static constexpr int K = 2;
  using C = Cx<T>;
  C* x; C* r; const C* p; const C* s; const C* t; const C* rt;
  C alpha, omega; int half;
  __device__ void load(const State* st) {
    alpha = fromd2<C>(st->alpha); omega = fromd2<C>(st->omega); half = st->half;
  }
  __device__ void operator()(int64_t i, double2* acc) {
    if (half) { x[i] = caxpy(x[i], alpha, p[i]); return; }
    // every load issued before the first store (the pointers are not
    // restrict-qualified, so a store would otherwise order the loads after it)
    const C xi = x[i], pi = p[i], si = s[i], ti = t[i], rti = rt[i];
    x[i] = caxpy(caxpy(xi, alpha, pi), omega, si);
    const C ri = caxmy(si, omega, ti);
    r[i] = ri;
    nrm_acc(acc[0], ri);
    dotc_acc(acc[1], rti, ri);
  }
  static __device__ void finish(State* st, const double2* sm) {
    const int k = st->iter + 1;
    if (st->half) {
      push_hist(st, k, st->ss);
      set_done(st, ST_CONVERGED, k);
      return;
    }
    bool stop;
    conv_check_common(st, k, sm[0].x, stop);
    if (stop) return;
    const double2 rho_new = sm[1];
    if (!zfinite(rho_new)) { set_done(st, ST_NONFINITE, k); return; }
    if (zzero(rho_new)) { set_done(st, ST_BREAKDOWN, k, BD_RHO); return; }
    st->beta = zmul(zdiv(rho_new, st->rho), zdiv(st->alpha, st->omega));
    st->rho = rho_new;
    st->iter = k;
  }
};

// ---- BiCGSTAB with the X and P passes merged (single GPU, stencil / SELL
// SpMV; Engine::bs_merge_ok, CCG_BS_MERGE=1).  ρ' = ⟨r̃, r'⟩ with r' = s − ωt
// is linear in r', so the t = A s product, which already reduces ⟨t,s⟩ and
// ⟨t,t⟩, also reduces ⟨r̃,s⟩ and ⟨r̃,t⟩ and its scalar step forms
// ρ' = ⟨r̃,s⟩ − ω⟨r̃,t⟩ and β right after ω.  The x / r update and the next
// direction p = r' + β(p − ωv) are then ONE pass (5 vectors read, 3 written)
// instead of BsX (5 + 2) followed by BsP (3 + 1): 4 launches and 16 instead of
// 19 vector streams per iteration.  Same recurrence in exact arithmetic; ρ'
// differs from the directly summed ⟨r̃, r'⟩ by rounding (a cancellation of
// relative size ‖s‖/‖r'‖), so this path is compared with the oracle by the
// P-envelope, not bit for bit with the default path.  The ρ' = 0 / non-finite
// tests stay where the literal recurrence has them — after the convergence
// test of the merged pass.
template <typename T>
struct BsTm {   // t = A s ; ⟨t,s⟩, ⟨t,t⟩, ⟨r̃,s⟩, ⟨r̃,t⟩ ; ω, ρ', β
  static constexpr int K = 4;
  using C = Cx<T>;
  C* t; const C* s; const C* rt;
  __device__ void load(const State*) {}
  using Pre = C;   // early load of r̃ (matvec.cuh EpiPre)
  __device__ Pre pre(int64_t i) const { return rt[i]; }
  // the stencil passes the product's own input element (s, by construction of bicgstab_iter's
  // merged path: single GPU, no preconditioner) from its register instead of a second load
  static constexpr bool WANTS_X = true;
  __device__ void post_x(int64_t i, C val, Pre rti, C si, double2* acc) {
    t[i] = val;
    dotc_acc(acc[0], val, si);
    nrm_acc(acc[1], val);
    dotc_acc(acc[2], rti, si);
    dotc_acc(acc[3], rti, val);
  }
  __device__ void post(int64_t i, C val, Pre rti, double2* acc) { post_x(i, val, rti, s[i], acc); }
  __device__ void operator()(int64_t i, C val, double2* acc) { post(i, val, pre(i), acc); }
  static __device__ void finish(State* st, const double2* sm) {
    BsT<T>::finish(st, sm);
    if (st->done) return;
    const double2 wt = zmul(st->omega, sm[3]);
    const double2 rho_new = make_double2(sm[2].x - wt.x, sm[2].y - wt.y);
    st->pb_rho = rho_new;   // tested in BsXP::finish, after the convergence test
    st->beta = zmul(zdiv(rho_new, st->rho), zdiv(st->alpha, st->omega));
  }
};

template <typename T>
struct BsXP {   // x += αp + ωs ; r = s − ωt ; p = r + β(p − ωv) ; ‖r‖²   (half-step: x += αp)
  static constexpr int K = 1;
  using C = Cx<T>;
  C* x; C* r; C* p; const C* s; const C* t; const C* v;
  C alpha, omega, beta; int half;
  __device__ void load(const State* st) {
    alpha = fromd2<C>(st->alpha); omega = fromd2<C>(st->omega); beta = fromd2<C>(st->beta); half = st->half;
  }
  __device__ void operator()(int64_t i, double2* acc) {
    if (half) { x[i] = caxpy(x[i], alpha, p[i]); return; }
    const C xi = x[i], pi = p[i], si = s[i], ti = t[i], vi = v[i];
    x[i] = caxpy(caxpy(xi, alpha, pi), omega, si);
    const C ri = caxmy(si, omega, ti);
    r[i] = ri;
    p[i] = bs_pnew(ri, pi, vi, beta, omega, 0);
    nrm_acc(acc[0], ri);
  }
  static __device__ void finish(State* st, const double2* sm) {
    const int k = st->iter + 1;
    if (st->half) {
      push_hist(st, k, st->ss);
      set_done(st, ST_CONVERGED, k);
      return;
    }
    bool stop;
    conv_check_common(st, k, sm[0].x, stop);
    if (stop) return;
    const double2 rho_new = st->pb_rho;
    if (!zfinite(rho_new)) { set_done(st, ST_NONFINITE, k); return; }
    if (zzero(rho_new)) { set_done(st, ST_BREAKDOWN, k, BD_RHO); return; }
    st->rho = rho_new;
    st->iter = k;
  }
};

// ===========================================================================
// O2 CGNE (Craig).  Setup: AH r → P0 (π, α).  Per iteration:
// [A p → r −= αAp, x += αp, ‖r‖²] → [Aᴴ r → p = Aᴴr + βp, ‖p‖²]
// ===========================================================================
__device__ __forceinline__ void cgne_pi(State* st, double pi) {
  const int k = st->iter + 1;
  st->matvecs_ah++;
  if (pi == 0.0) { set_done(st, ST_BREAKDOWN, k - 1, BD_PI); return; }
  st->pi_r = pi;
  st->alpha_r = st->rho_r / pi;
  if (!isfinite(st->alpha_r)) { set_done(st, ST_NONFINITE, k - 1); return; }
}

template <typename T>
struct CgP0 {  // p = Aᴴ r (setup)
  static constexpr int K = 1;
  using C = Cx<T>;
  C* p;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C w, double2* acc) { p[i] = w; nrm_acc(acc[0], w); }
  static __device__ void finish(State* st, const double2* s) { cgne_pi(st, s[0].x); }
};

template <typename T>
struct CgP {  // p = Aᴴ r + βp
  static constexpr int K = 1;
  using C = Cx<T>;
  C* p;
  T beta;
  __device__ void load(const State* st) { beta = (T)st->beta_r; }
  __device__ void operator()(int64_t i, C w, double2* acc) {
    C pi = p[i];
    C v; v.x = w.x + beta * pi.x; v.y = w.y + beta * pi.y;
    p[i] = v;
    nrm_acc(acc[0], v);
  }
  static __device__ void finish(State* st, const double2* s) { cgne_pi(st, s[0].x); }
};

template <typename T>
struct CgQ {  // r −= α(Ap) ; x += αp ; ‖r‖²
  static constexpr int K = 1;
  using C = Cx<T>;
  C* r; C* x; const C* p;
  T alpha;
  __device__ void load(const State* st) { alpha = (T)st->alpha_r; }
  __device__ void operator()(int64_t i, C q, double2* acc) {
    C pi = p[i], xi = x[i], ri = r[i];
    xi.x += alpha * pi.x; xi.y += alpha * pi.y;
    ri.x -= alpha * q.x; ri.y -= alpha * q.y;
    x[i] = xi; r[i] = ri;
    nrm_acc(acc[0], ri);
  }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter + 1;
    st->matvecs_a++;
    bool stop;
    conv_check_common(st, k, s[0].x, stop);
    if (stop) return;
    st->beta_r = s[0].x / st->rho_r;
    st->rho_r = s[0].x;
    st->iter = k;
  }
};

// ===========================================================================
// O3 QMR (no look-ahead, Aᴴ form).  Setup: V.  Per iteration:
// P → [A p → p̃, ε] → [Aᴴ q → w̃, ṽ, ‖ṽ‖², ‖w̃‖²] → DV (d, s, x, r, ‖r‖², v, w, δ)
// ===========================================================================
__device__ __forceinline__ void qmr_delta(State* st, double2 delta) {
  // start of iteration k = iter + 1
  const int k = st->iter + 1;
  if (st->rnrm == 0.0) { set_done(st, ST_BREAKDOWN, k - 1, BD_VNORM); return; }
  if (st->xnrm == 0.0) { set_done(st, ST_BREAKDOWN, k - 1, BD_WNORM); return; }
  if (!zfinite(delta)) { set_done(st, ST_NONFINITE, k - 1); return; }
  if (zzero(delta)) { set_done(st, ST_BREAKDOWN, k - 1, BD_DELTA); return; }
  st->delta = delta;
  if (st->iter > 0) {
    st->cp = zdiv(zscal(delta, st->xnrm), st->eps);             // ξδ/ε
    st->cq = zconj(zdiv(zscal(delta, st->rnrm), st->eps));      // conj(ρδ/ε)
  }
}

template <typename T>
struct QmV {  // v = ṽ/ρ ; w = w̃/ξ ; δ = ⟨w, v⟩   (setup)
  static constexpr int K = 1;
  using C = Cx<T>;
  const C* vt; const C* wt; C* v; C* w;
  T rn, xn;
  __device__ void load(const State* st) { rn = (T)st->rnrm; xn = (T)st->xnrm; }
  __device__ void operator()(int64_t i, double2* acc) {
    const C vi = cdivr(vt[i], rn), wi = cdivr(wt[i], xn);
    v[i] = vi; w[i] = wi;
    dotc_acc(acc[0], wi, vi);
  }
  static __device__ void finish(State* st, const double2* s) { qmr_delta(st, s[0]); }
};

template <typename T>
struct QmP {  // p = v − (ξδ/ε)p ; q = w − conj(ρδ/ε)q   (k=1: p = v, q = w)
  static constexpr int K = 0;
  using C = Cx<T>;
  const C* v; const C* w; C* p; C* q;
  C cp, cq; int first;
  __device__ void load(const State* st) {
    first = st->iter == 0; cp = fromd2<C>(st->cp); cq = fromd2<C>(st->cq);
  }
  __device__ void operator()(int64_t i, double2*) {
    if (first) { const C vi = v[i], wi = w[i]; p[i] = vi; q[i] = wi; return; }
    const C vi = v[i], pi = p[i], wi = w[i], qi = q[i];
    p[i] = caxmy(vi, cp, pi);
    q[i] = caxmy(wi, cq, qi);
  }
  static __device__ void finish(State*, const double2*) {}
};

template <typename T>
struct QmPt {  // p̃ = A p ; ε = ⟨q, p̃⟩ ; β = ε/δ
  static constexpr int K = 1;
  using C = Cx<T>;
  C* pt; const C* q;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C val, double2* acc) { const C b = q[i]; pt[i] = val; dotc_acc(acc[0], b, val); }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter + 1;
    st->matvecs_a++;
    const double2 eps = s[0];
    if (!zfinite(eps)) { set_done(st, ST_NONFINITE, k - 1); return; }
    if (zzero(eps)) { set_done(st, ST_BREAKDOWN, k - 1, BD_EPSILON); return; }
    st->eps = eps;
    st->beta = zdiv(eps, st->delta);
    if (zzero(st->beta)) { set_done(st, ST_BREAKDOWN, k - 1, BD_BETA); return; }
  }
};

template <typename T>
struct QmVW {  // w̃ = Aᴴq − conj(β)w ; ṽ = p̃ − βv ; ‖ṽ‖², ‖w̃‖² ; θ, γ, η
  static constexpr int K = 2;
  using C = Cx<T>;
  C* vt; C* wt; const C* pt; const C* v; const C* w;
  C beta, cbeta;
  __device__ void load(const State* st) { beta = fromd2<C>(st->beta); cbeta = fromd2<C>(zconj(st->beta)); }
  __device__ void operator()(int64_t i, C u, double2* acc) {
    const C wti = caxmy(u, cbeta, w[i]);
    const C vti = caxmy(pt[i], beta, v[i]);
    wt[i] = wti; vt[i] = vti;
    nrm_acc(acc[0], vti);
    nrm_acc(acc[1], wti);
  }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter + 1;
    st->matvecs_ah++;
    const double rn = sqrt(s[0].x), xn = sqrt(s[1].x);
    st->rnrm_next = rn; st->xnrm_next = xn;
    const double theta = rn / (st->gamma_prev * zabs(st->beta));
    const double gamma = 1.0 / sqrt(1.0 + theta * theta);
    if (!isfinite(theta) || !isfinite(gamma)) { set_done(st, ST_NONFINITE, k - 1); return; }
    if (gamma == 0.0) { set_done(st, ST_BREAKDOWN, k - 1, BD_GAMMA); return; }
    // η = −η ρ γ² / (β γ_prev²)
    const double2 num = zscal(zscal(zscal(zscal(st->eta, -1.0), st->rnrm), gamma), gamma);
    const double2 den = zscal(zscal(st->beta, st->gamma_prev), st->gamma_prev);
    st->eta = zdiv(num, den);
    st->theta = theta; st->gamma = gamma;
    const double tg = st->theta_prev * gamma;
    st->c2 = tg * tg;
  }
};

template <typename T>
struct QmDV {  // d, s ; x += d ; r −= s ; ‖r‖² ; v = ṽ/ρ' ; w = w̃/ξ' ; δ' = ⟨w, v⟩
  static constexpr int K = 2;
  using C = Cx<T>;
  C* d; C* sv; C* x; C* r; const C* p; const C* pt;
  const C* vt; const C* wt; C* v; C* w;
  C eta; T c2, rn, xn; int first;
  __device__ void load(const State* st) {
    eta = fromd2<C>(st->eta); c2 = (T)st->c2; rn = (T)st->rnrm_next; xn = (T)st->xnrm_next;
    first = st->iter == 0;
  }
  __device__ void operator()(int64_t i, double2* acc) {
    const C pi = p[i], pti = pt[i], xi = x[i], rold = r[i], vti = vt[i], wti = wt[i];
    C dd = czero<C>(), ss = czero<C>();
    if (!first) { dd = d[i]; ss = sv[i]; }
    C di = cmul(eta, pi), si = cmul(eta, pti);
    if (!first) {
      di.x += c2 * dd.x; di.y += c2 * dd.y;
      si.x += c2 * ss.x; si.y += c2 * ss.y;
    }
    d[i] = di; sv[i] = si;
    x[i] = cadd(xi, di);
    const C ri = csub(rold, si);
    r[i] = ri;
    nrm_acc(acc[0], ri);
    const C vi = cdivr(vti, rn), wi = cdivr(wti, xn);
    v[i] = vi; w[i] = wi;
    dotc_acc(acc[1], wi, vi);
  }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter + 1;
    bool stop;
    conv_check_common(st, k, s[0].x, stop);
    if (stop) return;
    st->rnrm = st->rnrm_next; st->xnrm = st->xnrm_next;
    st->gamma_prev = st->gamma; st->theta_prev = st->theta;
    st->iter = k;
    qmr_delta(st, s[1]);
  }
};

// ===========================================================================
// O4 BiCOR.  Per iteration: [A r → r̂, ρ = ⟨r*, r̂⟩] → P → [Aᴴ p* → q*, ξ = ⟨q*, q⟩] → X
// ===========================================================================
__device__ __forceinline__ void rho_step(State* st, double2 rho, bool count_a) {
  const int k = st->iter + 1;
  if (count_a) st->matvecs_a++;
  if (!zfinite(rho)) { set_done(st, ST_NONFINITE, k - 1); return; }
  if (zzero(rho)) { set_done(st, ST_BREAKDOWN, k - 1, BD_RHO); return; }
  st->rho = rho;
  if (st->iter > 0) st->beta = zdiv(rho, st->rho_prev);
}
__device__ __forceinline__ void xi_step(State* st, double2 xi) {
  const int k = st->iter + 1;
  if (zzero(xi)) { set_done(st, ST_BREAKDOWN, k - 1, BD_XI); return; }
  st->alpha = zdiv(st->rho, xi);
  if (!zfinite(st->alpha)) { set_done(st, ST_NONFINITE, k - 1); return; }
}
__device__ __forceinline__ void r_step(State* st, double rr) {
  const int k = st->iter + 1;
  bool stop;
  conv_check_common(st, k, rr, stop);
  if (stop) return;
  st->rho_prev = st->rho;
  st->iter = k;
}

template <typename T>
struct RhoEpi {  // r̂ = A r ; ρ = ⟨shadow, r̂⟩   (BiCOR and CORS)
  static constexpr int K = 1;
  using C = Cx<T>;
  C* rh; const C* sh;
  __device__ void load(const State*) {}
  // early load of the epilogue input (issued with the product's loads; matvec.cuh EpiPre)
  using Pre = C;
  __device__ Pre pre(int64_t i) const { return sh[i]; }
  __device__ void post(int64_t i, C val, Pre b, double2* acc) { rh[i] = val; dotc_acc(acc[0], b, val); }
  __device__ void operator()(int64_t i, C val, double2* acc) { post(i, val, pre(i), acc); }
  static __device__ void finish(State* st, const double2* s) { rho_step(st, s[0], true); }
};

template <typename T>
struct BcP {  // p = r + βp ; p* = r* + conj(β)p* ; q = r̂ + βq   (k=1: copies)
  static constexpr int K = 0;
  using C = Cx<T>;
  const C* r; const C* rs; const C* rh; C* p; C* ps; C* q;
  C beta, cbeta; int first;
  __device__ void load(const State* st) {
    first = st->iter == 0; beta = fromd2<C>(st->beta); cbeta = fromd2<C>(zconj(st->beta));
  }
  __device__ void operator()(int64_t i, double2*) {
    const C ri = r[i], rsi = rs[i], rhi = rh[i];
    if (first) { p[i] = ri; ps[i] = rsi; q[i] = rhi; return; }
    const C pi = p[i], psi = ps[i], qi = q[i];
    p[i] = caxpy(ri, beta, pi);
    ps[i] = caxpy(rsi, cbeta, psi);
    q[i] = caxpy(rhi, beta, qi);
  }
  static __device__ void finish(State*, const double2*) {}
};

template <typename T>
struct BcQs {  // q* = Aᴴ p* ; ξ = ⟨q*, q⟩ ; α = ρ/ξ
  static constexpr int K = 1;
  using C = Cx<T>;
  C* qs; const C* q;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C w, double2* acc) { qs[i] = w; dotc_acc(acc[0], w, q[i]); }
  static __device__ void finish(State* st, const double2* s) { st->matvecs_ah++; xi_step(st, s[0]); }
};

template <typename T>
struct BcX {  // x += αp ; r −= αq ; r* −= conj(α)q* ; ‖r‖²
  static constexpr int K = 1;
  using C = Cx<T>;
  C* x; C* r; C* rs; const C* p; const C* q; const C* qs;
  C alpha, calpha;
  __device__ void load(const State* st) { alpha = fromd2<C>(st->alpha); calpha = fromd2<C>(zconj(st->alpha)); }
  __device__ void operator()(int64_t i, double2* acc) {
    const C xi = x[i], pi = p[i], rold = r[i], qi = q[i], rsi = rs[i], qsi = qs[i];
    x[i] = caxpy(xi, alpha, pi);
    const C ri = caxmy(rold, alpha, qi);
    r[i] = ri;
    rs[i] = caxmy(rsi, calpha, qsi);
    nrm_acc(acc[0], ri);
  }
  static __device__ void finish(State* st, const double2* s) { r_step(st, s[0].x); }
};

// ===========================================================================
// O5 CORS (transpose-free).  Per iteration:
// [A r → r̂, ρ = ⟨r₀*, r̂⟩] → P (e, ê, q̂) → [A q̂ → q, ξ = ⟨r₀*, q⟩] → H (h, ĥ, x, r, ‖r‖²)
// ===========================================================================
template <typename T>
struct CoP {  // e = r + βh ; ê = r̂ + βĥ ; q̂ = ê + β(ĥ + βq̂)   (k=1: e = r, ê = q̂ = r̂)
  static constexpr int K = 0;
  using C = Cx<T>;
  const C* r; const C* rh; const C* h; const C* hh; C* e; C* eh; C* qh;
  C beta; int first;
  __device__ void load(const State* st) { first = st->iter == 0; beta = fromd2<C>(st->beta); }
  __device__ void operator()(int64_t i, double2*) {
    if (first) { const C v = rh[i], ri = r[i]; e[i] = ri; eh[i] = v; qh[i] = v; return; }
    const C hhi = hh[i], ri = r[i], hi = h[i], rhi = rh[i], qhi = qh[i];
    e[i] = caxpy(ri, beta, hi);
    const C ehi = caxpy(rhi, beta, hhi);
    eh[i] = ehi;
    qh[i] = caxpy(ehi, beta, caxpy(hhi, beta, qhi));
  }
  static __device__ void finish(State*, const double2*) {}
};

template <typename T>
struct CoQ {  // q = A q̂ ; ξ = ⟨r₀*, q⟩ ; α = ρ/ξ
  static constexpr int K = 1;
  using C = Cx<T>;
  C* q; const C* r0s;
  __device__ void load(const State*) {}
  // early load of the epilogue input (issued with the product's loads; matvec.cuh EpiPre)
  using Pre = C;
  __device__ Pre pre(int64_t i) const { return r0s[i]; }
  __device__ void post(int64_t i, C val, Pre b, double2* acc) { q[i] = val; dotc_acc(acc[0], b, val); }
  __device__ void operator()(int64_t i, C val, double2* acc) { post(i, val, pre(i), acc); }
  static __device__ void finish(State* st, const double2* s) { st->matvecs_a++; xi_step(st, s[0]); }
};

template <typename T>
struct CoH {  // h = e − αq̂ ; ĥ = ê − αq ; x += α(e + h) ; r −= α(ê + ĥ) ; ‖r‖²
  static constexpr int K = 1;
  using C = Cx<T>;
  const C* e; const C* eh; const C* qh; const C* q; C* h; C* hh; C* x; C* r;
  C alpha;
  __device__ void load(const State* st) { alpha = fromd2<C>(st->alpha); }
  __device__ void operator()(int64_t i, double2* acc) {
    const C ei = e[i], ehi = eh[i], qhi = qh[i], qi = q[i], xi = x[i], rold = r[i];
    const C hi = caxmy(ei, alpha, qhi);
    const C hhi = caxmy(ehi, alpha, qi);
    h[i] = hi; hh[i] = hhi;
    x[i] = caxpy(xi, alpha, cadd(ei, hi));
    const C ri = caxmy(rold, alpha, cadd(ehi, hhi));
    r[i] = ri;
    nrm_acc(acc[0], ri);
  }
  static __device__ void finish(State* st, const double2* s) { r_step(st, s[0].x); }
};

// ===========================================================================
// BiCG, CGS, CGNR (§2.1), COCR (§3.4) on the
// same matvec engine and fused passes (recurrences restated in DESIGN.md §2).
// ===========================================================================
// ρ' = ⟨r̃, r⟩ read at the end of an iteration (BiCG, CGS): after the
// convergence test; zero → BREAKDOWN(rho) with k completed (the oracle raises
// at the top of iteration k+1).
__device__ __forceinline__ void next_rho(State* st, int k, double rr, double2 rho_new) {
  bool stop;
  conv_check_common(st, k, rr, stop);
  if (stop) return;
  if (!zfinite(rho_new)) { set_done(st, ST_NONFINITE, k); return; }
  if (zzero(rho_new)) { set_done(st, ST_BREAKDOWN, k, BD_RHO); return; }
  st->beta = zdiv(rho_new, st->rho);
  st->rho = rho_new;
  st->iter = k;
}
__device__ __forceinline__ void sigma_step(State* st, double2 sigma) {
  const int k = st->iter + 1;
  if (zzero(sigma)) { set_done(st, ST_BREAKDOWN, k - 1, BD_SIGMA); return; }
  st->alpha = zdiv(st->rho, sigma);
  if (!zfinite(st->alpha)) { set_done(st, ST_NONFINITE, k - 1); return; }
}

// ---- BiCG.  P → [A p → q, σ = ⟨p̃, q⟩ ; Aᴴ p̃ → q̃] → X
template <typename T>
struct BgP {  // p = r + βp ; p̃ = r̃ + conj(β)p̃   (k=1: copies)
  static constexpr int K = 0;
  using C = Cx<T>;
  const C* r; const C* rt; C* p; C* pt;
  C beta, cbeta; int first;
  __device__ void load(const State* st) {
    first = st->iter == 0; beta = fromd2<C>(st->beta); cbeta = fromd2<C>(zconj(st->beta));
  }
  __device__ void operator()(int64_t i, double2*) {
    const C ri = r[i], rti = rt[i];
    if (first) { p[i] = ri; pt[i] = rti; return; }
    const C pi = p[i], pti = pt[i];
    p[i] = caxpy(ri, beta, pi);
    pt[i] = caxpy(rti, cbeta, pti);
  }
  static __device__ void finish(State*, const double2*) {}
};

template <typename T>
struct BgQ {  // q = A p ; σ = ⟨p̃, q⟩ ; α = ρ/σ   (counts the paired Aᴴp̃ too)
  static constexpr int K = 1;
  using C = Cx<T>;
  C* q; const C* pt;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C val, double2* acc) { const C b = pt[i]; q[i] = val; dotc_acc(acc[0], b, val); }
  static __device__ void finish(State* st, const double2* s) {
    st->matvecs_a++;
    st->matvecs_ah++;
    sigma_step(st, s[0]);
  }
};

template <typename T>
struct BgX {  // x += αp ; r −= αq ; r̃ −= conj(α)q̃ ; ‖r‖², ⟨r̃, r⟩
  static constexpr int K = 2;
  using C = Cx<T>;
  C* x; C* r; C* rt; const C* p; const C* q; const C* qt;
  C alpha, calpha;
  __device__ void load(const State* st) { alpha = fromd2<C>(st->alpha); calpha = fromd2<C>(zconj(st->alpha)); }
  __device__ void operator()(int64_t i, double2* acc) {
    const C xi = x[i], pi = p[i], rold = r[i], qi = q[i], rtold = rt[i], qti = qt[i];
    x[i] = caxpy(xi, alpha, pi);
    const C ri = caxmy(rold, alpha, qi);
    const C rti = caxmy(rtold, calpha, qti);
    r[i] = ri; rt[i] = rti;
    nrm_acc(acc[0], ri);
    dotc_acc(acc[1], rti, ri);
  }
  static __device__ void finish(State* st, const double2* s) { next_rho(st, st->iter + 1, s[0].x, s[1]); }
};

// ---- CGS.  P → [A p → v, σ = ⟨r̃, v⟩] → Q → [A(u+q) → r −= α·, ‖r‖², ⟨r̃, r⟩]
template <typename T>
struct CsP {  // u = r + βq ; p = u + β(q + βp)   (k=1: u = p = r)
  static constexpr int K = 0;
  using C = Cx<T>;
  const C* r; const C* q; C* p; C* u;
  C beta; int first;
  __device__ void load(const State* st) { first = st->iter == 0; beta = fromd2<C>(st->beta); }
  __device__ void operator()(int64_t i, double2*) {
    if (first) { const C ri = r[i]; u[i] = ri; p[i] = ri; return; }
    const C qi = q[i], ri = r[i], pi = p[i];
    const C ui = caxpy(ri, beta, qi);
    u[i] = ui;
    p[i] = caxpy(ui, beta, caxpy(qi, beta, pi));
  }
  static __device__ void finish(State*, const double2*) {}
};

template <typename T>
struct CsV {  // v = A p ; σ = ⟨r̃, v⟩ ; α = ρ/σ
  static constexpr int K = 1;
  using C = Cx<T>;
  C* v; const C* rt;
  __device__ void load(const State*) {}
  // early load of the epilogue input (issued with the product's loads; matvec.cuh EpiPre)
  using Pre = C;
  __device__ Pre pre(int64_t i) const { return rt[i]; }
  __device__ void post(int64_t i, C val, Pre b, double2* acc) { v[i] = val; dotc_acc(acc[0], b, val); }
  __device__ void operator()(int64_t i, C val, double2* acc) { post(i, val, pre(i), acc); }
  static __device__ void finish(State* st, const double2* s) { st->matvecs_a++; sigma_step(st, s[0]); }
};

template <typename T>
struct CsQ {  // q = u − αv ; u + q ; x += α(u + q)
  static constexpr int K = 0;
  using C = Cx<T>;
  const C* u; const C* v; C* q; C* uq; C* x;
  C alpha;
  __device__ void load(const State* st) { alpha = fromd2<C>(st->alpha); }
  __device__ void operator()(int64_t i, double2*) {
    const C ui = u[i], vi = v[i], xi = x[i];
    const C qi = caxmy(ui, alpha, vi);
    q[i] = qi;
    const C s = cadd(ui, qi);
    uq[i] = s;
    x[i] = caxpy(xi, alpha, s);
  }
  static __device__ void finish(State*, const double2*) {}
};

template <typename T>
struct CsR {  // r −= α A(u + q) ; ‖r‖², ⟨r̃, r⟩
  static constexpr int K = 2;
  using C = Cx<T>;
  C* r; const C* rt;
  C alpha;
  __device__ void load(const State* st) { alpha = fromd2<C>(st->alpha); }
  struct Pre { C r, rt; };   // early loads (matvec.cuh EpiPre)
  __device__ Pre pre(int64_t i) const { return Pre{r[i], rt[i]}; }
  __device__ void post(int64_t i, C w, Pre q, double2* acc) {
    const C ri = caxmy(q.r, alpha, w);
    r[i] = ri;
    nrm_acc(acc[0], ri);
    dotc_acc(acc[1], q.rt, ri);
  }
  __device__ void operator()(int64_t i, C w, double2* acc) { post(i, w, pre(i), acc); }
  static __device__ void finish(State* st, const double2* s) {
    st->matvecs_a++;
    next_rho(st, st->iter + 1, s[0].x, s[1]);
  }
};

// ---- COCR (complex-symmetric A; unconjugated [u, v]).  Setup: [A r → Ar, μ].
// Per iteration: P ([Ap, Ap] → α) → X (x, r, ‖r‖²) → [A r → Ar, μ' → β]
template <typename T>
struct CrAr0 {  // setup: Ar = A r₀ ; μ = [r₀, Ar₀]
  static constexpr int K = 1;
  using C = Cx<T>;
  C* ar; const C* r;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C val, double2* acc) { const C b = r[i]; ar[i] = val; dotu_acc(acc[0], b, val); }
  static __device__ void finish(State* st, const double2* s) { st->matvecs_a++; st->rho = s[0]; }
};

template <typename T>
struct CrAr {  // Ar = A r ; μ' = [r, Ar] ; β = μ'/μ   (end of iteration k = iter)
  static constexpr int K = 1;
  using C = Cx<T>;
  C* ar; const C* r;
  __device__ void load(const State*) {}
  // early load of the epilogue input (issued with the product's loads; matvec.cuh EpiPre)
  using Pre = C;
  __device__ Pre pre(int64_t i) const { return r[i]; }
  __host__ __device__ const void* pre_src() const { return r; }   // the product's own input (EpiPreSrc)
  __device__ void post(int64_t i, C val, Pre b, double2* acc) { ar[i] = val; dotu_acc(acc[0], b, val); }
  __device__ void operator()(int64_t i, C val, double2* acc) { post(i, val, pre(i), acc); }
  static __device__ void finish(State* st, const double2* s) {
    st->matvecs_a++;
    const int kc = st->iter - 1;   // the oracle raises inside iteration iter
    if (zzero(st->rho)) { set_done(st, ST_BREAKDOWN, kc, BD_RHO); return; }
    st->beta = zdiv(s[0], st->rho);
    if (!zfinite(st->beta)) { set_done(st, ST_NONFINITE, kc); return; }
    st->rho = s[0];
  }
};

template <typename T>
struct CrP {  // p = r + βp ; Ap = Ar + βAp (k=1: copies) ; [Ap, Ap] ; α = μ/[Ap, Ap]
  static constexpr int K = 1;
  using C = Cx<T>;
  const C* r; const C* ar; C* p; C* ap;
  C beta; int first;
  __device__ void load(const State* st) { first = st->iter == 0; beta = fromd2<C>(st->beta); }
  __device__ void operator()(int64_t i, double2* acc) {
    C pi, api;
    if (first) { pi = r[i]; api = ar[i]; }
    else { pi = caxpy(r[i], beta, p[i]); api = caxpy(ar[i], beta, ap[i]); }
    p[i] = pi; ap[i] = api;
    dotu_acc(acc[0], api, api);
  }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter + 1;
    if (zzero(s[0])) { set_done(st, ST_BREAKDOWN, k - 1, BD_XI); return; }
    st->alpha = zdiv(st->rho, s[0]);
    if (!zfinite(st->alpha)) { set_done(st, ST_NONFINITE, k - 1); return; }
  }
};

template <typename T>
struct CrX {  // x += αp ; r −= αAp ; ‖r‖²
  static constexpr int K = 1;
  using C = Cx<T>;
  C* x; C* r; const C* p; const C* ap;
  C alpha;
  __device__ void load(const State* st) { alpha = fromd2<C>(st->alpha); }
  __device__ void operator()(int64_t i, double2* acc) {
    const C xi = x[i], pi = p[i], rold = r[i], api = ap[i];
    x[i] = caxpy(xi, alpha, pi);
    const C ri = caxmy(rold, alpha, api);
    r[i] = ri;
    nrm_acc(acc[0], ri);
  }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter + 1;
    bool stop;
    conv_check_common(st, k, s[0].x, stop);
    if (stop) return;
    st->iter = k;
  }
};

// ---- CGNR (CG on AᴴA x = Aᴴy).  Setup: [Aᴴ r → p = z, γ].  Per iteration:
// [A p → w, ‖w‖² → α] → X (x, r, ‖r‖²) → [Aᴴ r → z, γ' → β] → P (p = z + βp)
template <typename T>
struct CnZ0 {  // setup: p = z = Aᴴ r₀ ; γ = ‖z‖²
  static constexpr int K = 1;
  using C = Cx<T>;
  C* p;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C w, double2* acc) { p[i] = w; nrm_acc(acc[0], w); }
  static __device__ void finish(State* st, const double2* s) { st->matvecs_ah++; st->rho_r = s[0].x; }
};

template <typename T>
struct CnW {  // w = A p ; α = γ/‖w‖²
  static constexpr int K = 1;
  using C = Cx<T>;
  C* w;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C val, double2* acc) { w[i] = val; nrm_acc(acc[0], val); }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter + 1;
    st->matvecs_a++;
    if (s[0].x == 0.0) { set_done(st, ST_BREAKDOWN, k - 1, BD_PI); return; }
    st->alpha_r = st->rho_r / s[0].x;
    if (!isfinite(st->alpha_r)) { set_done(st, ST_NONFINITE, k - 1); return; }
  }
};

template <typename T>
struct CnX {  // x += αp ; r −= αw ; ‖r‖²
  static constexpr int K = 1;
  using C = Cx<T>;
  C* x; C* r; const C* p; const C* w;
  T alpha;
  __device__ void load(const State* st) { alpha = (T)st->alpha_r; }
  __device__ void operator()(int64_t i, double2* acc) {
    C xi = x[i], ri = r[i];
    const C pi = p[i], wi = w[i];
    xi.x += alpha * pi.x; xi.y += alpha * pi.y;
    ri.x -= alpha * wi.x; ri.y -= alpha * wi.y;
    x[i] = xi; r[i] = ri;
    nrm_acc(acc[0], ri);
  }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter + 1;
    bool stop;
    conv_check_common(st, k, s[0].x, stop);
    if (stop) return;
    st->iter = k;
  }
};

template <typename T>
struct CnZ {  // z = Aᴴ r ; γ' = ‖z‖² ; β = γ'/γ
  static constexpr int K = 1;
  using C = Cx<T>;
  C* z;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C w, double2* acc) { z[i] = w; nrm_acc(acc[0], w); }
  static __device__ void finish(State* st, const double2* s) {
    st->matvecs_ah++;
    st->beta_r = s[0].x / st->rho_r;
    st->rho_r = s[0].x;
  }
};

template <typename T>
struct CnP {  // p = z + βp
  static constexpr int K = 0;
  using C = Cx<T>;
  const C* z; C* p;
  T beta;
  __device__ void load(const State* st) { beta = (T)st->beta_r; }
  __device__ void operator()(int64_t i, double2*) {
    const C zi = z[i], pi = p[i];
    C v; v.x = zi.x + beta * pi.x; v.y = zi.y + beta * pi.y;
    p[i] = v;
  }
  static __device__ void finish(State*, const double2*) {}
};

// ---- TFQMR (§2.1; Saad Alg. 7.8 in pairs of half-steps, readings R9-R11).
// Setup: [A u₀ → v = A u₀, σ → α].  Pair k: E (pass, first half-step) →
// [A u₂ → O: second half-step, ρ', β] (skipped after an E exit) → U (pass:
// pending x update; u = w + βu₂) → [A u → v = Au + β(Au₂ + βv), σ → α]
__device__ __forceinline__ bool tf_step(State* st, double ww, int bound_mult) {
  // θ, c, τ, η from ‖w_{m+1}‖²; returns true on convergence (τ²·(m+2) ≤ tol²‖r₀‖²)
  const double theta = sqrt(ww) / st->tau;
  const double c = 1.0 / sqrt(1.0 + theta * theta);
  const double tau = st->tau * theta * c;
  const double2 eta = zscal(st->alpha, c * c);
  const int k = st->iter + 1;
  if (!isfinite(theta) || !isfinite(tau) || !zfinite(eta)) { set_done(st, ST_NONFINITE, k - 1); return false; }
  st->theta = theta; st->tau = tau; st->eta = eta;
  const double bound2 = tau * tau * (double)bound_mult;
  if (bound2 <= st->tol2r0) { push_hist(st, k, bound2); return true; }
  st->ss = bound2;
  return false;
}

template <typename T>
struct TfV0 {  // setup: v = A u₀ (= A u_even) ; σ = ⟨r₀*, v⟩ ; α = ρ/σ
  static constexpr int K = 1;
  using C = Cx<T>;
  C* v; C* aue; const C* rs;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C val, double2* acc) { const C b = rs[i]; v[i] = val; aue[i] = val; dotc_acc(acc[0], b, val); }
  static __device__ void finish(State* st, const double2* s) { st->matvecs_a++; sigma_step(st, s[0]); }
};

template <typename T>
struct TfE {  // u₂ = u − αv ; w −= α·A u ; d = u + (θ²η/α)d ; ‖w‖² → θ, c, τ, η
  static constexpr int K = 1;
  using C = Cx<T>;
  const C* u; const C* v; const C* aue; C* u2; C* w; C* d;
  C alpha, coef; int first;
  __device__ void load(const State* st) {
    first = st->iter == 0;
    alpha = fromd2<C>(st->alpha);
    coef = fromd2<C>(zdiv(zscal(st->eta, st->theta * st->theta), st->alpha));
  }
  __device__ void operator()(int64_t i, double2* acc) {
    const C ui = u[i], vi = v[i], wold = w[i], auei = aue[i];
    const C dold = first ? ui : d[i];
    u2[i] = caxmy(ui, alpha, vi);
    const C wi = caxmy(wold, alpha, auei);
    w[i] = wi;
    d[i] = first ? ui : caxpy(ui, coef, dold);
    nrm_acc(acc[0], wi);
  }
  static __device__ void finish(State* st, const double2* s) {
    if (tf_step(st, s[0].x, 2 * (st->iter + 1))) { st->half = 1; st->gate2 = 1; }
  }
};

template <typename T>
struct TfO {  // A u₂ ; x += η d (E's update) ; w −= α A u₂ ; d = u₂ + (θ²η/α)d ; ‖w‖², ⟨r₀*, w⟩
  static constexpr int K = 2;
  using C = Cx<T>;
  C* au; C* x; C* w; C* d; const C* u2; const C* rs;
  C alpha, eta, coef;
  __device__ void load(const State* st) {
    alpha = fromd2<C>(st->alpha);
    eta = fromd2<C>(st->eta);
    coef = fromd2<C>(zdiv(zscal(st->eta, st->theta * st->theta), st->alpha));
  }
  __device__ void operator()(int64_t i, C val, double2* acc) {
    const C di = d[i], xi = x[i], wold = w[i], u2i = u2[i], rsi = rs[i];
    au[i] = val;
    x[i] = caxpy(xi, eta, di);
    const C wi = caxmy(wold, alpha, val);
    w[i] = wi;
    d[i] = caxpy(u2i, coef, di);
    nrm_acc(acc[0], wi);
    dotc_acc(acc[1], rsi, wi);
  }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter + 1;
    st->matvecs_a++;
    if (tf_step(st, s[0].x, 2 * k + 1)) { st->fin = 1; return; }
    if (st->done) return;
    if (k >= st->maxit) return;                       // R2: no products for an iterate nobody uses
    const double2 rho_new = s[1];
    if (!zfinite(rho_new)) { set_done(st, ST_NONFINITE, k - 1); return; }
    if (zzero(rho_new)) { set_done(st, ST_BREAKDOWN, k - 1, BD_RHO); return; }
    st->beta = zdiv(rho_new, st->rho);
    st->rho = rho_new;
  }
};

template <typename T>
struct TfU {  // x += η d (the pending update) ; u = w + β u₂ ; end of pair k
  static constexpr int K = 1;
  using C = Cx<T>;
  C* x; const C* d; const C* w; const C* u2; C* u;
  C eta, beta; int stop;
  __device__ void load(const State* st) {
    eta = fromd2<C>(st->eta); beta = fromd2<C>(st->beta);
    stop = st->half || st->fin || st->iter + 1 >= st->maxit;
  }
  __device__ void operator()(int64_t i, double2*) {
    const C xi = x[i], di = d[i];
    C wi = czero<C>(), u2i = czero<C>();
    if (!stop) { wi = w[i]; u2i = u2[i]; }
    x[i] = caxpy(xi, eta, di);
    if (!stop) u[i] = caxpy(wi, beta, u2i);
  }
  static __device__ void finish(State* st, const double2*) {
    const int k = st->iter + 1;
    if (st->half || st->fin) { set_done(st, ST_CONVERGED, k); return; }
    push_hist(st, k, st->ss);
    st->iter = k;
    if (k >= st->maxit) set_done(st, ST_MAXIT, k);
  }
};

template <typename T>
struct TfV {  // A u (kept) ; v = A u + β(A u₂ + βv) ; σ = ⟨r₀*, v⟩ ; α = ρ/σ
  static constexpr int K = 1;
  using C = Cx<T>;
  C* aue; const C* au; C* v; const C* rs;
  C beta;
  __device__ void load(const State* st) { beta = fromd2<C>(st->beta); }
  __device__ void operator()(int64_t i, C val, double2* acc) {
    const C aui = au[i], vold = v[i], rsi = rs[i];
    aue[i] = val;
    const C vi = caxpy(val, beta, caxpy(aui, beta, vold));
    v[i] = vi;
    dotc_acc(acc[0], rsi, vi);
  }
  static __device__ void finish(State* st, const double2* s) {
    st->matvecs_a++;
    const double2 sigma = s[0];
    const int kc = st->iter - 1;            // the oracle raises inside pair `iter`
    if (zzero(sigma)) { set_done(st, ST_BREAKDOWN, kc, BD_SIGMA); return; }
    st->alpha = zdiv(st->rho, sigma);
    if (!zfinite(st->alpha)) { set_done(st, ST_NONFINITE, kc); return; }
  }
};

// ---- BiCGstab(ℓ) (§3.1; vanilla Sleijpen–Fokkema, readings R16-R18).
// Per BiCG step j: P_j (û_i = r̂_i − βû_i, i ≤ j) → [A û_j → û_{j+1}, γ → α] →
// X_j (r̂_i −= αû_{i+1}, x += αû₀, ‖r̂₀‖²) → [A r̂_j → r̂_{j+1}, ρ₁ → β].
// MR part: Gram pass (Z, z, and the ℓ×ℓ solve in its scalar step) → M (x, r̂₀,
// û₀ updates, ‖r̂₀‖², ⟨r̃, r̂₀⟩ → the next cycle's ρ₀, ρ₁, β).
constexpr int BL_MAX = 4;

template <typename T>
struct BlP {
  static constexpr int K = 0;
  using C = Cx<T>;
  C* u[BL_MAX + 1]; const C* r[BL_MAX + 1]; int J;
  C beta;
  __device__ void load(const State* st) { beta = fromd2<C>(st->beta); }
  __device__ void operator()(int64_t i, double2*) {
    for (int a = 0; a <= J; ++a) u[a][i] = caxmy(r[a][i], beta, u[a][i]);
  }
  static __device__ void finish(State*, const double2*) {}
};

template <typename T>
struct BlU {  // û_{j+1} = A û_j ; γ = ⟨r̃, û_{j+1}⟩ ; α = ρ₀/γ
  static constexpr int K = 1;
  using C = Cx<T>;
  C* un; const C* rt;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C val, double2* acc) { const C b = rt[i]; un[i] = val; dotc_acc(acc[0], b, val); }
  static __device__ void finish(State* st, const double2* s) { st->matvecs_a++; sigma_step(st, s[0]); }
};

template <typename T>
struct BlX {  // r̂_i −= α û_{i+1} (i ≤ j) ; x += α û₀ ; ‖r̂₀‖² ; stopping test
  static constexpr int K = 1;
  using C = Cx<T>;
  C* r[BL_MAX + 1]; const C* u[BL_MAX + 1]; C* x; int J;
  C alpha;
  __device__ void load(const State* st) { alpha = fromd2<C>(st->alpha); }
  __device__ void operator()(int64_t i, double2* acc) {
    for (int a = 0; a <= J; ++a) r[a][i] = caxmy(r[a][i], alpha, u[a + 1][i]);
    x[i] = caxpy(x[i], alpha, u[0][i]);
    nrm_acc(acc[0], r[0][i]);
  }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter + 1;
    const double rr = s[0].x;
    if (!isfinite(rr)) { set_done(st, ST_NONFINITE, k - 1); return; }
    push_hist(st, k, rr);
    st->iter = k;
    if (rr <= st->tol2r0) { set_done(st, ST_CONVERGED, k); return; }
    if (k >= st->maxit && (k % st->bl_l) != 0) set_done(st, ST_MAXIT, k);   // mid-cycle
  }
};

// ρ₁ → β for the next step (also the start of a cycle, after M)
__device__ __forceinline__ void bl_next_beta(State* st, double2 rho1) {
  const int k = st->iter;
  if (!zfinite(rho1)) { set_done(st, ST_NONFINITE, k); return; }
  if (zzero(st->rho)) { set_done(st, ST_BREAKDOWN, k, BD_RHO); return; }
  st->beta = zmul(st->alpha, zdiv(rho1, st->rho));
  st->rho = rho1;
}

template <typename T>
struct BlR {  // r̂_{j+1} = A r̂_j ; ρ₁ = ⟨r̃, r̂_{j+1}⟩ ; β = α ρ₁/ρ₀ (not the last step of a cycle)
  static constexpr int K = 1;
  using C = Cx<T>;
  C* rn; const C* rt;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C val, double2* acc) { const C b = rt[i]; rn[i] = val; dotc_acc(acc[0], b, val); }
  static __device__ void finish(State* st, const double2* s) { st->matvecs_a++; bl_next_beta(st, s[0]); }
};

template <typename T>
struct BlRL {  // r̂_ℓ = A r̂_{ℓ−1} (last step of a cycle: only the product)
  static constexpr int K = 1;
  using C = Cx<T>;
  C* rn;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C val, double2*) { rn[i] = val; }
  static __device__ void finish(State* st, const double2*) { st->matvecs_a++; }
};

// MR part, Gram pass: Z_ij = ⟨r̂_i, r̂_j⟩ (1 ≤ i ≤ j ≤ L), z_i = ⟨r̂_i, r̂₀⟩; the
// scalar step solves Z γ = z (partial pivoting by |·|², as the oracle) into the
// scratch gm->y and sets ω = γ_L.  Z lives in gm->R, z in gm->g.
template <typename T, int L>
struct BlGram {
  static constexpr int K = L * (L + 1) / 2 + L;
  using C = Cx<T>;
  const C* r[BL_MAX + 1];
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, double2* acc) {
    C v[L + 1];
#pragma unroll
    for (int a = 0; a <= L; ++a) v[a] = r[a][i];
    int p = 0;
#pragma unroll
    for (int a = 1; a <= L; ++a)
#pragma unroll
      for (int b = a; b <= L; ++b) dotc_acc(acc[p++], v[a], v[b]);
#pragma unroll
    for (int a = 1; a <= L; ++a) dotc_acc(acc[p++], v[a], v[0]);
  }
  static __device__ void finish(State* st, const double2* s) {
    GmDev* gm = reinterpret_cast<GmDev*>(st->gm);
    double2 M[L][L + 1];
    int p = 0;
    for (int a = 0; a < L; ++a)
      for (int b = a; b < L; ++b) { M[a][b] = s[p]; M[b][a] = zconj(s[p]); ++p; }
    for (int a = 0; a < L; ++a) M[a][L] = s[p++];
    for (int c = 0; c < L; ++c) {
      int piv = c;
      double best = M[c][c].x * M[c][c].x + M[c][c].y * M[c][c].y;
      for (int i = c + 1; i < L; ++i) {
        const double m2 = M[i][c].x * M[i][c].x + M[i][c].y * M[i][c].y;
        if (m2 > best) { best = m2; piv = i; }
      }
      if (zzero(M[piv][c])) { set_done(st, ST_BREAKDOWN, st->iter - 1, BD_OMEGA); return; }
      if (piv != c)
        for (int j = 0; j <= L; ++j) { const double2 t = M[c][j]; M[c][j] = M[piv][j]; M[piv][j] = t; }
      for (int i = c + 1; i < L; ++i) {
        const double2 f = zdiv(M[i][c], M[c][c]);
        for (int j = c; j <= L; ++j) {
          const double2 q = zmul(f, M[c][j]);
          M[i][j] = make_double2(M[i][j].x - q.x, M[i][j].y - q.y);
        }
      }
    }
    for (int i = L - 1; i >= 0; --i) {
      double2 t = M[i][L];
      for (int j = i + 1; j < L; ++j) {
        const double2 q = zmul(M[i][j], gm->y[j]);
        t = make_double2(t.x - q.x, t.y - q.y);
      }
      gm->y[i] = zdiv(t, M[i][i]);
      if (!zfinite(gm->y[i])) { set_done(st, ST_NONFINITE, st->iter - 1); return; }
    }
    st->omega = gm->y[L - 1];
  }
};

template <typename T, int L>
struct BlM {  // x += Σ γ_j r̂_{j−1} ; r̂₀ −= Σ γ_j r̂_j ; û₀ −= Σ γ_j û_j ; ‖r̂₀‖², ⟨r̃, r̂₀⟩
  static constexpr int K = 2;
  using C = Cx<T>;
  C* r[BL_MAX + 1]; C* u[BL_MAX + 1]; C* x; const C* rt;
  C g[L];
  __device__ void load(const State* st) {
    const GmDev* gm = reinterpret_cast<const GmDev*>(st->gm);
#pragma unroll
    for (int a = 0; a < L; ++a) g[a] = fromd2<C>(gm->y[a]);
  }
  __device__ void operator()(int64_t i, double2* acc) {
    C rv[L + 1];
#pragma unroll
    for (int a = 0; a <= L; ++a) rv[a] = r[a][i];
    C xv = x[i];
#pragma unroll
    for (int a = 1; a <= L; ++a) xv = caxpy(xv, g[a - 1], rv[a - 1]);
    x[i] = xv;
    C r0 = rv[0];
#pragma unroll
    for (int a = 1; a <= L; ++a) r0 = caxmy(r0, g[a - 1], rv[a]);
    r[0][i] = r0;
    C u0 = u[0][i];
#pragma unroll
    for (int a = 1; a <= L; ++a) u0 = caxmy(u0, g[a - 1], u[a][i]);
    u[0][i] = u0;
    nrm_acc(acc[0], r0);
    dotc_acc(acc[1], rt[i], r0);
  }
  static __device__ void finish(State* st, const double2* s) {
    const int k = st->iter;
    const double rr = s[0].x;
    if (!isfinite(rr)) { set_done(st, ST_NONFINITE, k - 1); return; }
    push_hist(st, k, rr);
    if (rr <= st->tol2r0) { set_done(st, ST_CONVERGED, k); return; }
    if (k >= st->maxit) { set_done(st, ST_MAXIT, k); return; }
    if (zzero(st->omega)) { set_done(st, ST_BREAKDOWN, k - 1, BD_OMEGA); return; }
    st->rho = zmul(make_double2(-st->omega.x, -st->omega.y), st->rho);   // ρ₀ = −ω ρ₀
    bl_next_beta(st, s[1]);
  }
};

// ---- pipelined BiCGSTAB (SURVEY §8(f) NEXT-2 iii; oracle _pbicgstab).
// Setup: [A r → w, σ → α] [A w → t].  Per iteration: P1 (p, s, z, q, y;
// ‖q‖², ⟨y,q⟩, ‖y‖² → half-step test, ω) → [A z → v] → P2 (x, r, w; ‖r‖²,
// ⟨r̃,r⟩, ⟨r̃,w⟩, ⟨r̃,s⟩, ⟨r̃,z⟩) → [A w → t; then β, α].
template <typename T>
struct PbW0 {  // setup: w₀ = A r₀ ; α₀ = ρ₀/⟨r̃, w₀⟩
  static constexpr int K = 1;
  using C = Cx<T>;
  C* w; const C* rt;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C val, double2* acc) { const C b = rt[i]; w[i] = val; dotc_acc(acc[0], b, val); }
  static __device__ void finish(State* st, const double2* s) { st->matvecs_a++; sigma_step(st, s[0]); }
};

template <typename T>
struct PbStore {  // a product stored (v = A z, t₀ = A w₀); counts it
  static constexpr int K = 1;
  using C = Cx<T>;
  C* out;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C val, double2*) { out[i] = val; }
  static __device__ void finish(State* st, const double2*) { st->matvecs_a++; }
};

template <typename T>
struct PbP1 {  // p, s, z updates ; q = r − αs ; y = w − αz ; ‖q‖², ⟨y,q⟩, ‖y‖²
  static constexpr int K = 3;
  using C = Cx<T>;
  const C* r; const C* w; const C* t; const C* v; C* p; C* s; C* z; C* q; C* y;
  C alpha, beta, omega; int first;
  __device__ void load(const State* st) {
    first = st->iter == 0;
    alpha = fromd2<C>(st->alpha); beta = fromd2<C>(st->beta); omega = fromd2<C>(st->omega);
  }
  __device__ void operator()(int64_t i, double2* acc) {
    C pi, si, zi;
    if (first) { pi = r[i]; si = w[i]; zi = t[i]; }
    else {
      pi = caxpy(r[i], beta, caxmy(p[i], omega, s[i]));
      si = caxpy(w[i], beta, caxmy(s[i], omega, z[i]));
      zi = caxpy(t[i], beta, caxmy(z[i], omega, v[i]));
    }
    const C ri = r[i], wi = w[i];
    p[i] = pi; s[i] = si; z[i] = zi;
    const C qi = caxmy(ri, alpha, si), yi = caxmy(wi, alpha, zi);
    q[i] = qi; y[i] = yi;
    nrm_acc(acc[0], qi);
    dotc_acc(acc[1], yi, qi);
    nrm_acc(acc[2], yi);
  }
  static __device__ void finish(State* st, const double2* sm) {
    const int k = st->iter + 1;
    const double qq = sm[0].x;
    if (!isfinite(qq)) { set_done(st, ST_NONFINITE, k - 1); return; }
    st->ss = qq;
    if (qq <= st->tol2r0) { st->half = 1; st->gate2 = 1; return; }
    const double yy = sm[2].x;
    if (yy == 0.0) { set_done(st, ST_BREAKDOWN, k - 1, BD_TT); return; }
    st->omega = make_double2(sm[1].x / yy, sm[1].y / yy);
    if (!zfinite(st->omega)) { set_done(st, ST_NONFINITE, k - 1); return; }
    if (zzero(st->omega)) { set_done(st, ST_BREAKDOWN, k - 1, BD_OMEGA); return; }
  }
};

template <typename T>
struct PbP2 {  // x += αp + ωq ; r = q − ωy ; w = y − ω(t − αv) ; ‖r‖², ⟨r̃,r⟩, ⟨r̃,w⟩, ⟨r̃,s⟩, ⟨r̃,z⟩
  static constexpr int K = 5;            // (half-step: x += αp only)
  using C = Cx<T>;
  C* x; C* r; C* w; const C* p; const C* q; const C* y; const C* t; const C* v; const C* s; const C* z;
  const C* rt;
  C alpha, omega; int half;
  __device__ void load(const State* st) {
    alpha = fromd2<C>(st->alpha); omega = fromd2<C>(st->omega); half = st->half;
  }
  __device__ void operator()(int64_t i, double2* acc) {
    if (half) { x[i] = caxpy(x[i], alpha, p[i]); return; }
    const C qi = q[i], yi = y[i], xi = x[i], pi = p[i], ti = t[i], vi = v[i];
    const C rti = rt[i], si = s[i], zi = z[i];
    x[i] = caxpy(caxpy(xi, alpha, pi), omega, qi);
    const C ri = caxmy(qi, omega, yi);
    const C wi = caxmy(yi, omega, caxmy(ti, alpha, vi));
    r[i] = ri; w[i] = wi;
    nrm_acc(acc[0], ri);
    dotc_acc(acc[1], rti, ri);
    dotc_acc(acc[2], rti, wi);
    dotc_acc(acc[3], rti, si);
    dotc_acc(acc[4], rti, zi);
  }
  static __device__ void finish(State* st, const double2* sm) {
    const int k = st->iter + 1;
    if (st->half) { push_hist(st, k, st->ss); set_done(st, ST_CONVERGED, k); return; }
    bool stop;
    conv_check_common(st, k, sm[0].x, stop);
    if (stop) return;
    st->pb_rho = sm[1]; st->pb_rw = sm[2]; st->pb_rs = sm[3]; st->pb_rz = sm[4];
    st->iter = k;
  }
};

template <typename T>
struct PbT {  // t = A w ; then β = (α/ω)(ρ'/ρ), α = ρ'/(⟨r̃,w⟩ + β⟨r̃,s⟩ − βω⟨r̃,z⟩)
  static constexpr int K = 1;
  using C = Cx<T>;
  C* t;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C val, double2*) { t[i] = val; }
  static __device__ void finish(State* st, const double2*) {
    st->matvecs_a++;
    const int kc = st->iter - 1;         // the oracle raises inside iteration `iter`
    const double2 rho_new = st->pb_rho;
    if (!zfinite(rho_new)) { set_done(st, ST_NONFINITE, kc); return; }
    if (zzero(rho_new)) { set_done(st, ST_BREAKDOWN, kc, BD_RHO); return; }
    const double2 beta = zmul(zdiv(st->alpha, st->omega), zdiv(rho_new, st->rho));
    st->beta = beta;
    st->rho = rho_new;
    const double2 bs = zmul(beta, st->pb_rs), bwz = zmul(zmul(beta, st->omega), st->pb_rz);
    const double2 den = make_double2(st->pb_rw.x + bs.x - bwz.x, st->pb_rw.y + bs.y - bwz.y);
    if (zzero(den)) { set_done(st, ST_BREAKDOWN, kc, BD_SIGMA); return; }
    st->alpha = zdiv(rho_new, den);
    if (!zfinite(st->alpha)) { set_done(st, ST_NONFINITE, kc); return; }
  }
};

// ---- right Jacobi preconditioning: B = A·D⁻¹
template <typename T>
struct JacScale {  // out = s ⊙ x  (product input D⁻¹x; x₀ → D x₀; exit x = D⁻¹u)
  static constexpr int K = 0;
  using C = Cx<T>;
  const C* x; const C* s; C* out;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, double2*) { out[i] = cmul(s[i], x[i]); }
  static __device__ void finish(State*, const double2*) {}
};

template <typename T, class Epi>
struct JacEpi {  // Bᴴv = conj(D⁻¹)(Aᴴv), Bᵀv = D⁻¹(Aᵀv): scale the product, then the method epilogue
  static constexpr int K = Epi::K;
  using C = Cx<T>;
  Epi epi;
  const C* dinv;   // at the output's index origin
  int conj;
  __device__ void load(const State* st) { epi.load(st); }
  __device__ void operator()(int64_t i, C val, double2* acc) {
    C s = dinv[i];
    if (conj) s.y = -s.y;
    epi(i, cmul(s, val), acc);
  }
  static __device__ void finish(State* st, const double2* sm) { Epi::finish(st, sm); }
};

}  // namespace ccg
