// gmres.cuh — restarted GMRES(m) (P:57 [§2.1] "rgmres").
//
// One Arnoldi step per replayed CUDA graph: w = A v_j (matvec engine), then
// classical Gram–Schmidt applied twice (CGS2, R13) as three passes
// of the tall-skinny kernel gm_pass over the basis V (nloc × (m+1), one
// vector per column block):
//   MODE 0: h  = Vᴴ w                       (multi-dot)
//   MODE 1: w −= V h ;  h₂ = Vᴴ w           (update fused with the next multi-dot)
//   MODE 2: w −= V h₂ ; ‖w‖²
// then a single-thread Givens step (gm_step), the normalisation of v_{j+1},
// and — gated by device flags, so the same graph serves every step — the
// cycle end (back substitution, x += V y) and the restart (r = y − A·x).
// Every reduction is a per-CTA fp64 partial summed in CTA order by the last
// CTA (deterministic); with world > 1 the rank sums are allgathered and
// summed in rank order.
#pragma once
#include "common.cuh"
#include "methods.cuh"

namespace ccg {

// MODE 0: out = Vᴴw ; MODE 1: w −= V·coef, out = Vᴴw ; MODE 2: w −= V·coef, out[0] = ‖w‖²
// FAST (default): the update's loads go in groups of 4 and a full tile's
// multi-dot loads are unrolled (issued before their FMAs).  Same operations
// in the same order; the compiler's FMA contraction of the unrolled code can
// differ at the last bit (config 5: identical iteration counts, true residual
// equal to 1e-17 relative).
template <typename T, int MODE, bool FAST = false>
__global__ void __launch_bounds__(GM_NT)
gm_pass(const typename CT<T>::c* __restrict__ V, int64_t ldv, typename CT<T>::c* __restrict__ w,
        const double2* __restrict__ coef, double2* out, int64_t nrows, const GmDev* gm, double2* part,
        unsigned* ticket, int fuse, const int* gate) {
  using C = typename CT<T>::c;
  constexpr int NW = GM_NT / 32;
  constexpr int NA = (GM_MAX + 1 + NW - 1) / NW;   // accumulators per lane (vectors per warp)
  if (pdl_gate(gate)) return;
  __shared__ C wt[GM_NT];
  __shared__ C cf[GM_MAX + 1];
  __shared__ double2 nsm[NW];
  __shared__ int am_last;
  const int J = gm->j + 1;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (MODE > 0)
    for (int i = t; i < J; i += GM_NT) cf[i] = fromd2<C>(coef[i]);
  double2 acc[NA];
#pragma unroll
  for (int a = 0; a < NA; ++a) acc[a] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int64_t base = (int64_t)blockIdx.x * GM_NT; base < nrows; base += (int64_t)gridDim.x * GM_NT) {
    const int64_t r = base + t;
    C wv = czero<C>();
    if (r < nrows) {
      wv = w[r];
      if (MODE > 0) {
        int i = 0;
        if constexpr (FAST) {
          for (; i + 4 <= J; i += 4) {
            C vv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) vv[u] = V[(int64_t)(i + u) * ldv + r];
#pragma unroll
            for (int u = 0; u < 4; ++u) wv = caxmy(wv, cf[i + u], vv[u]);
          }
        }
        for (; i < J; ++i) wv = caxmy(wv, cf[i], V[(int64_t)i * ldv + r]);
        w[r] = wv;
      }
    }
    if (MODE == 2) {
      nrm_acc(acc[0], wv);
    } else {
      __syncthreads();
      wt[t] = wv;
      __syncthreads();
      const int nr = (int)min((int64_t)GM_NT, nrows - base);
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        const int i = warp + a * NW;
        if (i < J) {
          const C* vi = V + (int64_t)i * ldv + base;
          if (FAST && nr == GM_NT) {
            C vv[GM_NT / 32];
#pragma unroll
            for (int k = 0; k < GM_NT / 32; ++k) vv[k] = vi[lane + 32 * k];
#pragma unroll
            for (int k = 0; k < GM_NT / 32; ++k) dotc_acc(acc[a], vv[k], wt[lane + 32 * k]);
          } else {
            for (int rr = lane; rr < nr; rr += 32) dotc_acc(acc[a], vi[rr], wt[rr]);
          }
        }
      }
    }
  }
  // per-CTA partials in fixed slots
  if (MODE == 2) {
    double2 v1[1] = {acc[0]};
    block_sum<1, GM_NT>(v1, nsm);
    if (t == 0) part[(size_t)blockIdx.x * (GM_MAX + 1)] = v1[0];
  } else {
#pragma unroll
    for (int a = 0; a < NA; ++a) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc[a].x += __shfl_xor_sync(0xffffffffu, acc[a].x, o);
        acc[a].y += __shfl_xor_sync(0xffffffffu, acc[a].y, o);
      }
      const int i = warp + a * NW;
      if (lane == 0 && i < J) part[(size_t)blockIdx.x * (GM_MAX + 1) + i] = acc[a];
    }
  }
  __syncthreads();
  if (t == 0) {
    __threadfence();
    am_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  const int nout = MODE == 2 ? 1 : J;
  for (int i = t; i < nout; i += GM_NT) {
    double2 s = make_double2(0.0, 0.0);
    for (unsigned c = 0; c < gridDim.x; ++c) {
      const double2 p = __ldcg(part + (size_t)c * (GM_MAX + 1) + i);
      s.x += p.x; s.y += p.y;
    }
    out[i] = s;                      // this rank's sum (fuse) or rank_sum slot (world > 1)
  }
  if (t == 0) *ticket = 0u;
  (void)fuse;
}

// world > 1: sum the allgathered rank sums in rank order
static __global__ void gm_ranksum(const double2* all, int world, int count, int stride, double2* out, const int* gate) {
  if (pdl_gate(gate)) return;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int r = 0; r < world; ++r) { s.x += all[r * stride + i].x; s.y += all[r * stride + i].y; }
    out[i] = s;
  }
}

// Arnoldi / Givens step (one thread)
static __global__ void gm_step(State* st, GmDev* gm, const int* gate) {
  if (pdl_gate(gate)) return;
  const int j = gm->j;
  const int k = ++gm->k;
  st->matvecs_a++;
  double2 h[GM_MAX + 1];
  for (int i = 0; i <= j; ++i) h[i] = make_double2(gm->hcol[i].x + gm->h2[i].x, gm->hcol[i].y + gm->h2[i].y);
  const double hn = sqrt(gm->ww2.x);
  bool fin = isfinite(hn);
  for (int i = 0; i <= j; ++i) fin = fin && zfinite(h[i]);
  if (!fin) { set_done(st, ST_NONFINITE, k - 1); gm->endflag = 1; return; }
  for (int i = 0; i < j; ++i) {                       // previous rotations
    const double2 a = h[i], b = h[i + 1];
    const double c = gm->cs[i];
    const double2 s = gm->sn[i];
    h[i] = make_double2(c * a.x + (s.x * b.x - s.y * b.y), c * a.y + (s.x * b.y + s.y * b.x));
    const double2 cs_ = zconj(s);
    h[i + 1] = make_double2(-(cs_.x * a.x - cs_.y * a.y) + c * b.x, -(cs_.x * a.y + cs_.y * a.x) + c * b.y);
  }
  const double2 a = h[j];                             // new rotation zeroing h_{j+1,j}
  double c;
  double2 s;
  if (zzero(a)) {
    c = 0.0; s = make_double2(1.0, 0.0);
  } else {
    const double aa = zabs(a);
    const double nu = sqrt(aa * aa + hn * hn);
    c = aa / nu;
    s = zscal(make_double2(a.x / aa, a.y / aa), hn / nu);
  }
  gm->cs[j] = c;
  gm->sn[j] = s;
  h[j] = make_double2(c * a.x + s.x * hn, c * a.y + s.y * hn);
  const double2 gj = gm->g[j];
  const double2 csn = zconj(s);
  gm->g[j + 1] = make_double2(-(csn.x * gj.x - csn.y * gj.y), -(csn.x * gj.y + csn.y * gj.x));
  gm->g[j] = zscal(gj, c);
  for (int i = 0; i <= j; ++i) gm->R[j * (GM_MAX + 1) + i] = h[i];
  const double res2 = gm->g[j + 1].x * gm->g[j + 1].x + gm->g[j + 1].y * gm->g[j + 1].y;
  push_hist(st, k, res2);
  st->iter = k;
  const bool conv = res2 <= st->tol2r0;
  if (conv || k >= st->maxit || j == gm->m - 1) {
    gm->endflag = 1;
    gm->noend = 0;
    gm->pend = conv ? ST_CONVERGED : (k >= st->maxit ? ST_MAXIT : -1);
  } else {
    gm->hn = hn;
    gm->j = j + 1;
  }
}

// v_{j+1} = w / h_{j+1,j} into the basis and the full-length product input
template <typename T>
__global__ void gm_normalize(typename CT<T>::c* V, int64_t ldv, const typename CT<T>::c* w,
                             typename CT<T>::c* full_slice, int64_t nrows, const GmDev* gm,
                             int use_beta, const int* gate) {
  using C = typename CT<T>::c;
  if (pdl_gate(gate)) return;
  const int jj = use_beta ? 0 : gm->j;
  const T d = (T)(use_beta ? gm->g[0].x : gm->hn);
  C* vj = V + (int64_t)jj * ldv;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const C v = cdivr(w[r], d);
    vj[r] = v;
    full_slice[r] = v;
  }
}

// back substitution R y = g (one thread); decides done / restart
static __global__ void gm_trisolve(State* st, GmDev* gm, const int* gate) {
  if (pdl_gate(gate)) return;
  const int J = gm->j + 1;
  for (int i = J - 1; i >= 0; --i) {
    double2 t = gm->g[i];
    for (int l = i + 1; l < J; ++l) {
      const double2 p = zmul(gm->R[l * (GM_MAX + 1) + i], gm->y[l]);
      t.x -= p.x; t.y -= p.y;
    }
    const double2 d = gm->R[i * (GM_MAX + 1) + i];
    if (zzero(d)) { set_done(st, ST_BREAKDOWN, gm->k - 1, BD_GAMMA); return; }
    gm->y[i] = zdiv(t, d);
    if (!zfinite(gm->y[i])) { set_done(st, ST_NONFINITE, gm->k - 1); return; }
  }
  gm->noxupd = 0;
  if (gm->pend >= 0) set_done(st, gm->pend, gm->k);
  else gm->norestart = 0;
}

// x += Σ_i y_i v_i (i in order)
template <typename T>
__global__ void gm_xupdate(typename CT<T>::c* __restrict__ x, const typename CT<T>::c* __restrict__ V, int64_t ldv,
                           int64_t nrows, const GmDev* gm, const int* gate) {
  using C = typename CT<T>::c;
  if (pdl_gate(gate)) return;
  const int J = gm->j + 1;
  __shared__ C ys[GM_MAX];
  for (int i = threadIdx.x; i < J; i += blockDim.x) ys[i] = fromd2<C>(gm->y[i]);
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    C xv = x[r];
    for (int i = 0; i < J; ++i) xv = caxpy(xv, ys[i], V[(int64_t)i * ldv + r]);
    x[r] = xv;
  }
}

// end of every replayed step: re-arm the flags
static __global__ void gm_reset(GmDev* gm) {
  pdl_wait();
  gm->endflag = 0;
  gm->noend = 1;
  gm->noxupd = 1;
  gm->norestart = 1;
}

// restart: r = y − A·x into v₀'s slot ; ‖r‖² → β, convergence, new cycle
template <typename T>
struct GmR {
  static constexpr int K = 1;
  using C = Cx<T>;
  const C* y; C* v0;
  __device__ void load(const State*) {}
  __device__ void operator()(int64_t i, C ax, double2* acc) {
    const C r = csub(y[i], ax);
    v0[i] = r;
    nrm_acc(acc[0], r);
  }
  static __device__ void finish(State* st, const double2* s) {
    GmDev* gm = reinterpret_cast<GmDev*>(st->gm);
    st->matvecs_a++;
    const double rr = s[0].x;
    if (!isfinite(rr)) { set_done(st, ST_NONFINITE, gm->k); return; }
    st->rr = rr;
    if (rr <= st->tol2r0) { set_done(st, ST_CONVERGED, gm->k); return; }
    gm->g[0] = make_double2(sqrt(rr), 0.0);
    gm->j = 0;
  }
};

}  // namespace ccg
