// cluster.cuh — the whole Krylov loop in ONE thread-block cluster (K8).
//
// Config 1 (n = 256, a 1 MiB matrix) is latency-bound (SURVEY §7 hard part 3,
// §8(d)): a graph-launched iteration is 4-6 dependent kernels of a few µs
// each.  Here one cluster of CL CTAs (up to 16, non-portable size) runs every
// iteration of a solve with no kernel boundary: CTA r owns rows
// [n·r/CL, n·(r+1)/CL) of A and of every vector; a phase (a fused vector pass
// or a product with its epilogue — the SAME functors as the multi-kernel path,
// methods.cuh) is followed by one cluster barrier (barrier.cluster arrive.release
// / wait.acquire: the vector writes of every CTA become visible to every
// other).  Reductions: each CTA's fp64 partials sit in its shared memory; after
// the barrier every CTA reads all CL partials over DSMEM and sums them in CTA
// order, so every CTA computes bit-identical sums and runs the phase's scalar
// step (finish) on its OWN shared-memory copy of the solver State —
// replicated, consistent by construction, no broadcast.  Control flow
// (done / gate2) is therefore uniform across the cluster.  CTA 0 writes the
// final State back.  Vectors written inside the kernel are read with plain
// (coherent) loads, never the read-only path.
#pragma once
#include "common.cuh"
#include "methods.cuh"

namespace ccg {

__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// read a double2 from the shared memory of CTA `cta` of this cluster
__device__ __forceinline__ double2 dsmem_ld(const double2* local_addr, unsigned cta) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local_addr)), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(cta));
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(ra) : "memory");
  return v;
}

constexpr int CL_NT = 512;
constexpr int CL_KMAX = 5;   // p-BiCGSTAB's second pass has 5 partial sums
constexpr int CL_MAX = 16;

template <typename T>
struct ClusterCtx {
  using C = typename CT<T>::c;
  State* st;            // this CTA's shared-memory copy
  double2 (*cpart)[CL_KMAX];   // [2][CL_KMAX] this CTA's phase sums (DSMEM-visible)
  double2* red_sm;      // block_sum scratch
  double2* all;         // [CL_MAX * CL_KMAX] gathered partials
  C* colsum;            // Aᴴ column partial scratch
  int buf;
  unsigned rank, CL;
  int64_t r0, r1, n, lda;
  const C* A;

  template <int K, class Fin>
  __device__ void reduce(double2 (&v)[K > 0 ? K : 1]) {
    if constexpr (K > 0) {
      block_sum<K, CL_NT>(v, red_sm);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) cpart[buf][k] = v[k];
      }
    }
    cl_sync();
    if constexpr (K > 0) {
      if (threadIdx.x < CL * K) all[threadIdx.x] = dsmem_ld(&cpart[buf][threadIdx.x % K], threadIdx.x / K);
      __syncthreads();
      if (threadIdx.x == 0) {
        double2 s[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          s[k] = make_double2(0.0, 0.0);
          for (unsigned c = 0; c < CL; ++c) { s[k].x += all[c * K + k].x; s[k].y += all[c * K + k].y; }
        }
        Fin::finish(st, s);
      }
      __syncthreads();
      buf ^= 1;
    }
  }

  // the same pass over ALL rows in every CTA, its sums over all rows formed
  // in-CTA (fixed order, identical in every CTA) and its scalar step run on the
  // CTA's own State: no barrier, no DSMEM.  Only for passes whose outputs do
  // not alias their inputs (every CTA writes the same values) and whose inputs
  // are complete (written by this CTA, or before the last barrier).
  template <class Op>
  __device__ void rpass(Op op) {
    constexpr int KK = Op::K > 0 ? Op::K : 1;
    op.load(st);
    double2 d[KK];
#pragma unroll
    for (int k = 0; k < KK; ++k) d[k] = make_double2(0.0, 0.0);
    for (int64_t i = threadIdx.x; i < n; i += CL_NT) op(i, d);
    if constexpr (Op::K > 0) {
      block_sum<Op::K, CL_NT>(d, red_sm);
      if (threadIdx.x == 0) Op::finish(st, d);
    }
    __syncthreads();
  }

  // fused vector pass over this CTA's rows
  template <class Op>
  __device__ void pass(Op op) {
    constexpr int KK = Op::K > 0 ? Op::K : 1;
    op.load(st);
    double2 d[KK];
#pragma unroll
    for (int k = 0; k < KK; ++k) d[k] = make_double2(0.0, 0.0);
    for (int64_t i = r0 + threadIdx.x; i < r1; i += CL_NT) op(i, d);
    reduce<Op::K, Op>(d);
  }

  // y_i = Σ_j A_ij x_j for this CTA's rows (warp per row), epilogue per row
  template <class Epi>
  __device__ void gemv(Epi epi, const C* x) {
    constexpr int KK = Epi::K > 0 ? Epi::K : 1;
    epi.load(st);
    double2 d[KK];
#pragma unroll
    for (int k = 0; k < KK; ++k) d[k] = make_double2(0.0, 0.0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t i = r0 + warp; i < r1; i += CL_NT / 32) {
      const C* a = A + i * lda;
      C acc = czero<C>();
      int64_t j = lane;
      for (; j + 32 * 7 < n; j += 32 * 8) {      // 8 independent loads in flight per lane
        C av[8], xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { av[u] = __ldg(a + j + 32 * u); xv[u] = x[j + 32 * u]; }
#pragma unroll
        for (int u = 0; u < 8; ++u) cfma(acc, av[u], xv[u]);
      }
      for (; j < n; j += 32) cfma(acc, __ldg(a + j), x[j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (lane == 0) epi(i, acc, d);
    }
    reduce<Epi::K, Epi>(d);
  }

  // y_j = Σ_i op(A_ij) x_i for this CTA's columns j ∈ [r0, r1) (A read once
  // over the cluster): thread = (column, row group), fixed-order group sum
  template <bool CONJ, class Epi>
  __device__ void gemvh(Epi epi, const C* x) {
    constexpr int KK = Epi::K > 0 ? Epi::K : 1;
    epi.load(st);
    double2 d[KK];
#pragma unroll
    for (int k = 0; k < KK; ++k) d[k] = make_double2(0.0, 0.0);
    const int ncol = (int)(r1 - r0);
    for (int c0 = 0; c0 < ncol; c0 += CL_NT) {
      const int w = min(CL_NT, ncol - c0);
      const int G = CL_NT / w;            // row groups
      const int c = threadIdx.x % w, g = threadIdx.x / w;
      C acc = czero<C>();
      if (g < G) {
        const int64_t j = r0 + c0 + c;
        int64_t i = g;
        for (; i + (int64_t)G * 7 < n; i += (int64_t)G * 8) {   // 8 independent loads in flight
          C av[8], xv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) { av[u] = __ldg(A + (i + (int64_t)G * u) * lda + j); xv[u] = x[i + (int64_t)G * u]; }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (CONJ) cfmac(acc, av[u], xv[u]); else cfma(acc, av[u], xv[u]);
          }
        }
        for (; i < n; i += G) {
          if (CONJ) cfmac(acc, __ldg(A + i * lda + j), x[i]); else cfma(acc, __ldg(A + i * lda + j), x[i]);
        }
        colsum[g * w + c] = acc;
      }
      __syncthreads();
      if (threadIdx.x < w) {
        C s = colsum[threadIdx.x];
        for (int gg = 1; gg < G; ++gg) s = cadd(s, colsum[gg * w + threadIdx.x]);
        epi(r0 + c0 + threadIdx.x, s, d);
      }
      __syncthreads();
    }
    reduce<Epi::K, Epi>(d);
  }
};

#define CL_PH(stmt) \
  if (!cx.st->done) { stmt; }

// ---- per-method iteration bodies (same phases as Engine::*_iter, world = 1)
template <typename T>
struct ClBicgstab {
  BsP<T> p; BsV<T> v; BsS<T> s; BsT<T> t; BsX<T> x;
  const typename CT<T>::c *pf, *sf;
  __device__ void setup(ClusterCtx<T>&) {}
  __device__ void iter(ClusterCtx<T>& cx) {
    CL_PH(cx.pass(p));
    CL_PH(cx.gemv(v, pf));
    CL_PH(cx.pass(s));
    if (!cx.st->gate2) cx.gemv(t, sf);
    CL_PH(cx.pass(x));
  }
};
// BiCGSTAB with 2 cluster barriers per iteration instead of 5: the P and S
// passes, the σ / ⟨t,s⟩,⟨t,t⟩ sums and the X pass run redundantly over all rows
// in every CTA (rpass); barriers only after each product (its rows come from
// every CTA).  P writes p out of place into the other of two buffers
// (iteration parity), so no CTA reads a p another CTA is overwriting; the X
// pass writes x only for this CTA's rows (x is updated in place), r for all
// rows.  Same arithmetic as the multi-kernel path, sums in another fixed order.
template <typename T>
struct BsPo {   // p_out = r (k = 1) | r + β(p_in − ωv)   (BsP out of place)
  static constexpr int K = 0;
  using C = Cx<T>;
  const C* r; const C* pin; C* pout; const C* v;
  C beta, omega; int first;
  __device__ void load(const State* st) {
    first = st->iter == 0;
    beta = fromd2<C>(st->beta); omega = fromd2<C>(st->omega);
  }
  __device__ void operator()(int64_t i, double2*) { pout[i] = bs_pnew(r[i], pin[i], v[i], beta, omega, first); }
  static __device__ void finish(State*, const double2*) {}
};
template <typename T>
struct BsXc {
  static constexpr int K = 2;
  using C = Cx<T>;
  BsX<T> b;
  int64_t r0, r1;
  __device__ void load(const State* st) { b.load(st); }
  __device__ void operator()(int64_t i, double2* acc) {
    const bool own = i >= r0 && i < r1;
    if (b.half) {
      if (own) b.x[i] = caxpy(b.x[i], b.alpha, b.p[i]);
      return;
    }
    const C si = b.s[i], ti = b.t[i], rti = b.rt[i];
    if (own) b.x[i] = caxpy(caxpy(b.x[i], b.alpha, b.p[i]), b.omega, si);   // BsX's arithmetic
    const C ri = caxmy(si, b.omega, ti);
    b.r[i] = ri;
    nrm_acc(acc[0], ri);
    dotc_acc(acc[1], rti, ri);
  }
  static __device__ void finish(State* st, const double2* sm) { BsX<T>::finish(st, sm); }
};
template <typename T>
struct ClBicgstabR {
  BsP<T> p; BsV<T> v; BsS<T> s; BsT<T> t; BsX<T> x;
  const typename CT<T>::c *pf, *sf;
  typename CT<T>::c* p2;   // the second p buffer
  __device__ void setup(ClusterCtx<T>&) {}
  __device__ void iter(ClusterCtx<T>& cx) {
    using C = typename CT<T>::c;
    C* pa = const_cast<C*>(pf);
    C* pin = (cx.st->iter & 1) ? p2 : pa;
    C* pout = (cx.st->iter & 1) ? pa : p2;
    CL_PH(cx.rpass(BsPo<T>{p.r, pin, pout, p.v}));       // p (all rows) into the other buffer
    CL_PH(cx.gemv(Store<T>{v.v}, pout));                  // own rows of v; barrier
    CL_PH(cx.rpass(EpiPass<C, BsV<T>>{v, v.v}));          // σ over all rows -> α
    CL_PH(cx.rpass(s));                                   // s (all rows), ‖s‖², half-step test
    if (!cx.st->gate2) {
      cx.gemv(Store<T>{t.t}, sf);                         // own rows of t; barrier
      cx.rpass(EpiPass<C, BsT<T>>{t, t.t});               // ⟨t,s⟩, ⟨t,t⟩ -> ω
    }
    BsX<T> xb = x;
    xb.p = pout;
    CL_PH(cx.rpass(BsXc<T>{xb, cx.r0, cx.r1}));
  }
};

template <typename T>
struct ClCgne {
  CgQ<T> q; CgP<T> p; CgP0<T> p0;
  const typename CT<T>::c *pf, *r;
  __device__ void setup(ClusterCtx<T>& cx) { cx.template gemvh<true>(p0, r); }
  __device__ void iter(ClusterCtx<T>& cx) {
    CL_PH(cx.gemv(q, pf));
    CL_PH(cx.template gemvh<true>(p, r));
  }
};
template <typename T>
struct ClQmr {
  QmP<T> p; QmPt<T> pt; QmVW<T> vw; QmDV<T> dv; QmV<T> v0;
  const typename CT<T>::c *pf, *q;
  __device__ void setup(ClusterCtx<T>& cx) { cx.pass(v0); }
  __device__ void iter(ClusterCtx<T>& cx) {
    CL_PH(cx.pass(p));
    CL_PH(cx.gemv(pt, pf));
    CL_PH(cx.template gemvh<true>(vw, q));
    CL_PH(cx.pass(dv));
  }
};
template <typename T>
struct ClBicor {
  RhoEpi<T> rho; BcP<T> p; BcQs<T> qs; BcX<T> x;
  const typename CT<T>::c *rf, *ps;
  __device__ void setup(ClusterCtx<T>&) {}
  __device__ void iter(ClusterCtx<T>& cx) {
    CL_PH(cx.gemv(rho, rf));
    CL_PH(cx.pass(p));
    CL_PH(cx.template gemvh<true>(qs, ps));
    CL_PH(cx.pass(x));
  }
};
template <typename T>
struct ClCors {
  RhoEpi<T> rho; CoP<T> p; CoQ<T> q; CoH<T> h;
  const typename CT<T>::c *rf, *qhf;
  __device__ void setup(ClusterCtx<T>&) {}
  __device__ void iter(ClusterCtx<T>& cx) {
    CL_PH(cx.gemv(rho, rf));
    CL_PH(cx.pass(p));
    CL_PH(cx.gemv(q, qhf));
    CL_PH(cx.pass(h));
  }
};
template <typename T>
struct ClBicg {
  BgP<T> p; BgQ<T> q; Store<T> qt; BgX<T> x;
  const typename CT<T>::c *pf, *pt;
  __device__ void setup(ClusterCtx<T>&) {}
  __device__ void iter(ClusterCtx<T>& cx) {
    CL_PH(cx.pass(p));
    CL_PH(cx.template gemvh<true>(qt, pt));   // q̃ = Aᴴp̃ first: BgQ's step counts both
    CL_PH(cx.gemv(q, pf));
    CL_PH(cx.pass(x));
  }
};
template <typename T>
struct ClCgs {
  CsP<T> p; CsV<T> v; CsQ<T> q; CsR<T> r;
  const typename CT<T>::c *pf, *uqf;
  __device__ void setup(ClusterCtx<T>&) {}
  __device__ void iter(ClusterCtx<T>& cx) {
    CL_PH(cx.pass(p));
    CL_PH(cx.gemv(v, pf));
    CL_PH(cx.pass(q));
    CL_PH(cx.gemv(r, uqf));
  }
};
template <typename T>
struct ClCocr {
  CrP<T> p; CrX<T> x; CrAr<T> ar; CrAr0<T> ar0;
  const typename CT<T>::c* rf;
  __device__ void setup(ClusterCtx<T>& cx) { cx.gemv(ar0, rf); }
  __device__ void iter(ClusterCtx<T>& cx) {
    CL_PH(cx.pass(p));
    CL_PH(cx.pass(x));
    CL_PH(cx.gemv(ar, rf));
  }
};
template <typename T>
struct ClCgnr {
  CnW<T> w; CnX<T> x; CnZ<T> z; CnP<T> p; CnZ0<T> z0;
  const typename CT<T>::c *pf, *r;
  __device__ void setup(ClusterCtx<T>& cx) { cx.template gemvh<true>(z0, r); }
  __device__ void iter(ClusterCtx<T>& cx) {
    CL_PH(cx.gemv(w, pf));
    CL_PH(cx.pass(x));
    CL_PH(cx.template gemvh<true>(z, r));
    CL_PH(cx.pass(p));
  }
};

// r₀ = y (or y − A·x₀) with its copies, and the exit true residual ‖y − A·x‖²
// (S:273-276): the phases ccg_solve runs around the iterations, done in-kernel
template <typename T>
struct ClCommon {
  InitR<T> ir;
  Copy<T> cp0;   // x₀ → full buffer (has_x0)
  Copy<T> cpx;   // x → full buffer (true residual)
  TrueRes<T> tr;
  const typename CT<T>::c* f2;
  int has_x0;
};

template <typename T>
struct ClTfqmr {
  TfE<T> e; TfO<T> o; TfU<T> u; TfV<T> v; TfV0<T> v0;
  const typename CT<T>::c *uf, *u2f;
  __device__ void setup(ClusterCtx<T>& cx) { cx.gemv(v0, uf); }
  __device__ void iter(ClusterCtx<T>& cx) {
    CL_PH(cx.pass(e));
    if (!cx.st->gate2) cx.gemv(o, u2f);
    CL_PH(cx.pass(u));
    CL_PH(cx.gemv(v, uf));
  }
};

// p-BiCGSTAB (NEXT-2 iii): same phases and buffers as the graph schedule
template <typename T>
struct ClPbicgstab {
  PbW0<T> w0; PbStore<T> t0; PbP1<T> p1; PbStore<T> v; PbP2<T> p2; PbT<T> t;
  const typename CT<T>::c *zf, *wf;
  __device__ void setup(ClusterCtx<T>& cx) {
    CL_PH(cx.gemv(w0, zf));
    CL_PH(cx.gemv(t0, wf));
  }
  __device__ void iter(ClusterCtx<T>& cx) {
    CL_PH(cx.pass(p1));
    if (!cx.st->gate2) cx.gemv(v, zf);
    CL_PH(cx.pass(p2));
    CL_PH(cx.gemv(t, wf));
  }
};

template <typename T, class M>
__global__ void __launch_bounds__(CL_NT, 1)
cluster_solve(M m, ClCommon<T> cm, State* gst, const typename CT<T>::c* __restrict__ A, int64_t lda, int64_t n) {
  using C = typename CT<T>::c;
  __shared__ State sst;
  __shared__ double2 cpart[2][CL_KMAX];
  __shared__ double2 red_sm[(CL_NT / 32) * CL_KMAX];
  __shared__ double2 all[CL_MAX * CL_KMAX];
  __shared__ C colsum[CL_NT];
  if (threadIdx.x == 0) sst = *gst;
  __syncthreads();
  ClusterCtx<T> cx;
  cx.st = &sst;
  cx.cpart = cpart;
  cx.red_sm = red_sm;
  cx.all = all;
  cx.colsum = colsum;
  cx.buf = 0;
  cx.rank = cl_rank();
  cx.CL = cl_size();
  cx.r0 = n * cx.rank / cx.CL;
  cx.r1 = n * (cx.rank + 1) / cx.CL;
  cx.n = n;
  cx.lda = lda;
  cx.A = A;
  cl_sync();                      // every CTA's shared memory is live before any DSMEM read
  if (cm.has_x0) {
    cx.pass(cm.cp0);
    cx.gemv(cm.ir, cm.f2);
  } else {
    cx.pass(cm.ir);
  }
  if (!sst.done) m.setup(cx);
  while (!sst.done) m.iter(cx);
  cx.pass(cm.cpx);
  cx.gemv(cm.tr, cm.f2);
  cl_sync();                      // no CTA exits while another may still read its partials
  if (cx.rank == 0 && threadIdx.x == 0) *gst = sst;
}

}  // namespace ccg
