// common.cuh — complex arithmetic, device state, deterministic reductions.
//
// Part of libccg.so (see include/ccg.h).  Nothing here is shared with the
// CPU oracle (oracle/), which is test infrastructure only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ccg {

// ---------------------------------------------------------------------------
// Programmatic dependent launch (sm_90+): every kernel of the path starts by
// waiting until its predecessor has completed and its writes are visible
// (pdl_gate / pdl_wait).  No kernel triggers early: griddepcontrol.wait only
// guarantees the writes made BEFORE the primary's trigger, and every kernel
// writes the State its successor gates on in its very last step, so the
// implicit trigger at exit is the only safe one; what PDL still buys is the
// successor's launch processing overlapping the predecessor's execution.
// A kernel launched without the PDL attribute passes the wait as a no-op.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ int pdl_gate(const int* gate) {
  pdl_wait();
  return *gate;
}

// ---------------------------------------------------------------------------
// complex types: cplx<float> = interleaved c64, cplx<double> = c128
// ---------------------------------------------------------------------------
template <typename T> struct CT;
template <> struct CT<float> {
  using c = float2;   // one complex
  using v = float4;   // 16-byte vector = 2 complex
  static constexpr int V = 2;
};
template <> struct CT<double> {
  using c = double2;
  using v = double2;  // 16-byte vector = 1 complex
  static constexpr int V = 1;
};

template <typename C> __device__ __forceinline__ C cmake(double re, double im) {
  C r; r.x = re; r.y = im; return r;
}
template <typename C> __device__ __forceinline__ C czero() { C r; r.x = 0; r.y = 0; return r; }
template <typename C> __device__ __forceinline__ C cadd(C a, C b) { C r; r.x = a.x + b.x; r.y = a.y + b.y; return r; }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { C r; r.x = a.x - b.x; r.y = a.y - b.y; return r; }
template <typename C> __device__ __forceinline__ C cconj(C a) { C r; r.x = a.x; r.y = -a.y; return r; }
// Real products that the compiler may not contract into an FMA (__fmul_rn /
// __dmul_rn): the vector updates below then round the same way in every
// kernel that inlines them, so a value formed in one kernel (a fused input
// transform, methods.cuh BsSIn) and recomputed in another (its epilogue) are
// the same bits — with plain `a*b - c*d` nvcc picks the contraction per call
// site.
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
  C r; r.x = rmul(a.x, b.x) - rmul(a.y, b.y); r.y = rmul(a.x, b.y) + rmul(a.y, b.x); return r;
}
// contractible product (FFT butterflies: no value there is recomputed elsewhere)
template <typename C> __device__ __forceinline__ C cmulc(C a, C b) {
  C r; r.x = a.x * b.x - a.y * b.y; r.y = a.x * b.y + a.y * b.x; return r;
}
// a + s*b
template <typename C> __device__ __forceinline__ C caxpy(C a, C s, C b) {
  C r;
  r.x = a.x + (rmul(s.x, b.x) - rmul(s.y, b.y));
  r.y = a.y + (rmul(s.x, b.y) + rmul(s.y, b.x));
  return r;
}
// a - s*b
template <typename C> __device__ __forceinline__ C caxmy(C a, C s, C b) {
  C r;
  r.x = a.x - (rmul(s.x, b.x) - rmul(s.y, b.y));
  r.y = a.y - (rmul(s.x, b.y) + rmul(s.y, b.x));
  return r;
}
// acc += a*b (4 FMAs)
template <typename C> __device__ __forceinline__ void cfma(C& acc, C a, C b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a)*b
template <typename C> __device__ __forceinline__ void cfmac(C& acc, C a, C b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y);
}
template <typename C> __device__ __forceinline__ C cscale(C a, double s) {
  C r; r.x = a.x * s; r.y = a.y * s; return r;
}
// complex / real (component-wise IEEE division)
template <typename C, typename R> __device__ __forceinline__ C cdivr(C a, R s) {
  C r; r.x = a.x / s; r.y = a.y / s; return r;
}
template <typename C> __device__ __forceinline__ double2 d2(C a) { return make_double2((double)a.x, (double)a.y); }
template <typename C> __device__ __forceinline__ C fromd2(double2 a) { C r; r.x = a.x; r.y = a.y; return r; }

// fp64 reduction helpers: acc += conj(a)*b, acc += |a|^2 (products formed in fp64)
template <typename C> __device__ __forceinline__ void dotc_acc(double2& acc, C a, C b) {
  double ax = a.x, ay = a.y, bx = b.x, by = b.y;
  acc.x = fma(ax, bx, acc.x); acc.x = fma(ay, by, acc.x);
  acc.y = fma(ax, by, acc.y); acc.y = fma(-ay, bx, acc.y);
}
// acc += a*b (unconjugated bilinear form [a, b], COCR)
template <typename C> __device__ __forceinline__ void dotu_acc(double2& acc, C a, C b) {
  double ax = a.x, ay = a.y, bx = b.x, by = b.y;
  acc.x = fma(ax, bx, acc.x); acc.x = fma(-ay, by, acc.x);
  acc.y = fma(ax, by, acc.y); acc.y = fma(ay, bx, acc.y);
}
template <typename C> __device__ __forceinline__ void nrm_acc(double2& acc, C a) {
  double ax = a.x, ay = a.y;
  acc.x = fma(ax, ax, acc.x); acc.x = fma(ay, ay, acc.x);
}

// fp64 complex scalar algebra (recurrence scalars)
__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 zdiv(double2 a, double2 b) {
  // Smith's algorithm
  if (fabs(b.x) >= fabs(b.y)) {
    double rr = b.y / b.x, den = b.x + b.y * rr;
    return make_double2((a.x + a.y * rr) / den, (a.y - a.x * rr) / den);
  } else {
    double rr = b.x / b.y, den = b.y + b.x * rr;
    return make_double2((a.x * rr + a.y) / den, (a.y * rr - a.x) / den);
  }
}
__device__ __forceinline__ double2 zconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 zscal(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double zabs(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ bool zfinite(double2 a) { return isfinite(a.x) && isfinite(a.y); }
__device__ __forceinline__ bool zzero(double2 a) { return a.x == 0.0 && a.y == 0.0; }

// ---------------------------------------------------------------------------
// GMRES(m) device workspace (gmres.cuh): Hessenberg/Givens data and the
// per-step flags that gate the cycle-end and restart kernels of the graph
// ---------------------------------------------------------------------------
constexpr int GM_MAX = 64;     // longest restart cycle
constexpr int GM_NT = 256;     // threads per CTA = rows per tile

struct GmDev {
  double2 hcol[GM_MAX + 1];               // pass-1 dots, then the rotated column
  double2 h2[GM_MAX + 1];                 // pass-2 dots
  double2 R[GM_MAX * (GM_MAX + 1)];       // rotated columns: R[j·(GM_MAX+1) + i]
  double2 g[GM_MAX + 1];
  double cs[GM_MAX];
  double2 sn[GM_MAX];
  double2 y[GM_MAX];
  double2 ww2;                            // ‖w‖² after the second pass (.x)
  double hn;                              // h_{j+1,j}
  int m, j, k;                            // restart length, inner index, Arnoldi steps
  int pend;                               // status to set after the x update (-1: restart)
  int endflag;                            // 1: cycle ended (skip the normalisation)
  int noend;                              // 0: run the cycle-end kernels
  int noxupd;                             // 0: run the x update
  int norestart;                          // 0: run the restart kernels
};


// ---------------------------------------------------------------------------
// Device-resident solver state.  Written only by single-thread "finish"
// steps; read by every kernel of the next phase (stream order).
// ---------------------------------------------------------------------------
struct State {
  int done;        // 1 => every gated kernel returns immediately
  int gate2;       // done || BiCGSTAB half-step exit (gates the 2nd matvec)
  int status;
  int iterations;
  int iter;        // completed iterations
  int maxit;
  int method;
  int half;        // BiCGSTAB half-step exit pending / taken
  int breakdown;
  int matvecs_a;
  int matvecs_ah;
  int hist_cap;
  double tol2;     // tol^2
  double r0sq;     // ‖r0‖^2
  double tol2r0;   // tol^2 ‖r0‖^2
  double rr;       // last ‖r‖^2 (or ‖s‖^2 at a half-step)
  double true_rr;  // ‖y − A x‖^2 at finalize
  double* hist;    // [hist_cap] ‖r_k‖/‖r0‖
  // recurrence scalars (fp64)
  double2 rho, rho_prev, alpha, omega, beta, delta, eps, eta, cp, cq;
  double rnrm, xnrm, rnrm_next, xnrm_next, gamma_prev, gamma, theta, theta_prev, c2;
  double rho_r, pi_r, alpha_r, beta_r;  // CGNE (real scalars)
  double tau;      // TFQMR τ_m
  void* gm;        // GmDev* (GMRES; BiCGstab(ℓ) scratch)
  int bl_l;        // BiCGstab(ℓ): ℓ
  double2 pb_rho, pb_rw, pb_rs, pb_rz;   // p-BiCGSTAB: ⟨r̃,r⟩, ⟨r̃,w⟩, ⟨r̃,s⟩, ⟨r̃,z⟩ of the last phase
  int fin;         // TFQMR: converged at the second half-step, x update pending
  double ss;
};

enum { ST_CONVERGED = 0, ST_MAXIT = 1, ST_BREAKDOWN = 2, ST_FALSE_CONV = 3, ST_NONFINITE = 4 };
enum { BD_NONE = 0, BD_RHO = 1, BD_SIGMA = 2, BD_TT = 3, BD_OMEGA = 4, BD_PI = 5, BD_DELTA = 6,
       BD_EPSILON = 7, BD_BETA = 8, BD_XI = 9, BD_VNORM = 10, BD_WNORM = 11, BD_GAMMA = 12 };
enum { M_BICGSTAB = 0, M_CGNE = 1, M_QMR = 2, M_BICOR = 3, M_CORS = 4,
       M_BICG = 5, M_CGS = 6, M_COCR = 7, M_CGNR = 8, M_TFQMR = 9, M_GMRES = 10,
       M_BICGSTABL = 11, M_PBICGSTAB = 12, M_COUNT = 13 };

__device__ __forceinline__ void set_done(State* st, int status, int iters, int bd = BD_NONE) {
  st->done = 1; st->gate2 = 1; st->status = status; st->iterations = iters; st->breakdown = bd;
}
__device__ __forceinline__ void push_hist(State* st, int k, double rr) {
  if (k < st->hist_cap && st->hist) st->hist[k] = st->r0sq > 0 ? sqrt(rr) / sqrt(st->r0sq) : 0.0;
  st->rr = rr;
}

// ---------------------------------------------------------------------------
// Deterministic two-level reduction: per-CTA partial in a fixed slot, the
// last CTA to finish (atomic ticket) sums the slots in slot order and either
// runs the phase's scalar step (single GPU) or stores this rank's sums for
// the scalar allgather (multi GPU).
// ---------------------------------------------------------------------------
struct Red {
  double2* part;      // [gridsize][K]
  unsigned* ticket;   // zero between launches
  double2* rank_sum;  // [K] (multi GPU)
  int fuse;           // 1 => run finish in the last CTA
};

template <int K, int NT>
__device__ __forceinline__ void block_sum(double2 (&v)[K], double2* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v[k].x += __shfl_xor_sync(0xffffffffu, v[k].x, o);
      v[k].y += __shfl_xor_sync(0xffffffffu, v[k].y, o);
    }
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sm[warp * K + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double2 s = make_double2(0.0, 0.0);
      for (int w = 0; w < NT / 32; ++w) { s.x += sm[w * K + k].x; s.y += sm[w * K + k].y; }
      v[k] = s;
    }
  }
}

__device__ __forceinline__ unsigned block_linear_id() {
  return blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
}
__device__ __forceinline__ unsigned grid_blocks() { return gridDim.x * gridDim.y * gridDim.z; }

// the CTA's K partial sums go to slot `bid` of `nb` (every slot written once
// per launch); the CTA that arrives last sums the slots in slot order
template <int K, int NT, class Fin>
__device__ __forceinline__ void finish_reduction_at(double2 (&v)[K], const Red& red, State* st, unsigned bid,
                                                    unsigned nb) {
  __shared__ double2 sm[(NT / 32) * K];
  __shared__ int am_last;
  block_sum<K, NT>(v, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) red.part[(size_t)bid * K + k] = v[k];
    __threadfence();
    unsigned t = atomicAdd(red.ticket, 1u);
    am_last = (t == nb - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double2 acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = make_double2(0.0, 0.0);
  // slots b = tid, tid + NT, … summed in that order; the loads of U slots are
  // issued together (one L2 round trip per U slots instead of one per slot —
  // this serial tail runs on one SM while the rest of the GPU waits)
  constexpr int U = K >= 8 ? 1 : 8 / K;   // <= 32 registers of loads in flight
  for (unsigned b0 = threadIdx.x; b0 < nb; b0 += U * NT) {
    double2 p[U][K];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned b = b0 + u * NT;
#pragma unroll
      for (int k = 0; k < K; ++k)
        p[u][k] = b < nb ? __ldcg(red.part + (size_t)b * K + k) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (b0 + u * NT < nb) {
#pragma unroll
        for (int k = 0; k < K; ++k) { acc[k].x += p[u][k].x; acc[k].y += p[u][k].y; }
      }
    }
  }
  block_sum<K, NT>(acc, sm);
  if (threadIdx.x == 0) {
    *red.ticket = 0u;
    if (red.fuse) {
      Fin::finish(st, acc);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) red.rank_sum[k] = acc[k];
    }
  }
}

template <int K, int NT, class Fin>
__device__ __forceinline__ void finish_reduction(double2 (&v)[K], const Red& red, State* st) {
  finish_reduction_at<K, NT, Fin>(v, red, st, block_linear_id(), grid_blocks());
}

}  // namespace ccg
