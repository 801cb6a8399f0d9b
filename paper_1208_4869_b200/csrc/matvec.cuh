// matvec.cuh — the matvec engine: dense A·x, dense Aᴴ·x / Aᵀ·x, CSR A·x.
//
// PAPER.md P:95 [§5]: "All the communication to matvec, cmatvec is set in
// module arraymodule" — matvec = A·x, cmatvec = Aᴴ·x.  All three
// kernels are HBM-bandwidth bound: A is streamed once with
// 128-bit loads and evict-first caching; the vector is kept in L2/L1.
//
// Epilogue functors (method phases, methods.cuh) receive each finished
// output element (row i, value) and accumulate up to K fp64 partial sums,
// which finish_reduction() turns into the phase's recurrence scalars.
#pragma once
#include <type_traits>
#include <utility>
#include "bulk.cuh"
#include "common.cuh"

namespace ccg {

// streaming 16-byte load (ld.global.cs: evict-first, A is touched once)
__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ float2 ld_stream(const float2* p) { return __ldcs(p); }

// ---------------------------------------------------------------------------
// L2 residency of part of A (DESIGN.md §4 "L2-resident rows"): a matrix a
// little larger than the 126 MB L2 (config 2: 268 MB) is re-read every
// product, so during a solve the rows with ((i >> 3) & 63) < pin (pin/64 of
// A, sized to ~80 MB) are loaded with an L2 evict_last policy and stay
// resident from one product to the next, the other rows evict-first.  The
// predicate takes groups of 8 consecutive rows, so every CTA's row range is
// pinned in the same proportion (no CTA waits on HBM while others hit L2).
// l2_demote() returns the lines to normal priority when the solve ends.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ bool row_pinned(int64_t i, int pin) { return (int)((i >> 3) & 63) < pin; }
__device__ __forceinline__ float4 ld_hint(const float4* p, uint64_t pol) {
  float4 v;
  asm("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld_hint(const double2* p, uint64_t pol) {
  double2 v;
  asm("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float2 ld_hint(const float2* p, uint64_t pol) {
  float2 v;
  asm("ld.global.L1::no_allocate.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
               : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
  return v;
}
// A-load functors: LdA streams (evict-first); LdPin picks the policy per row
struct LdA {
  template <class LV>
  __device__ __forceinline__ LV operator()(const LV* p, int64_t) const { return ld_stream(p); }
};
struct LdPin {
  uint64_t keep, drop;
  int pin;
  template <class LV>
  __device__ __forceinline__ LV operator()(const LV* p, int64_t row) const {
    return ld_hint(p, row_pinned(row, pin) ? keep : drop);
  }
};
__device__ __forceinline__ LdPin make_ldpin(int pin) { return LdPin{l2_policy_last(), l2_policy_first(), pin}; }

// demote the pinned rows of A to normal L2 priority (one thread per 128-B line)
template <typename T>
__global__ void l2_demote(const typename CT<T>::c* A, int64_t lda, int64_t nrows, int64_t n, int pin) {
  using C = typename CT<T>::c;
  const int64_t lines = (n * (int64_t)sizeof(C) + 127) / 128 + 1;   // +1: row starts need not be 128-B aligned
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nrows * lines;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / lines;
    if (!row_pinned(i, pin)) continue;
    const uintptr_t row = reinterpret_cast<uintptr_t>(A + i * lda) & ~(uintptr_t)127;
    const char* p = reinterpret_cast<const char*>(row) + (k % lines) * 128;
    // the extra line of an aligned row starts at or past the row's end — for
    // the last row that is past the end of A (an unmapped address when A ends
    // its allocation: intermittent illegal access with every row pinned)
    if (p >= reinterpret_cast<const char*>(A + i * lda + n)) continue;
    asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(p));
  }
}

// unpack a 16-byte vector into V complex values
__device__ __forceinline__ void unpack(const float4& v, float2 (&c)[2]) {
  c[0] = make_float2(v.x, v.y); c[1] = make_float2(v.z, v.w);
}
__device__ __forceinline__ void unpack(const double2& v, double2 (&c)[1]) { c[0] = v; }
__device__ __forceinline__ void unpack(const float2& v, float2 (&c)[1]) { c[0] = v; }

// ---------------------------------------------------------------------------
// Early epilogue loads.  An epilogue that reads other vectors at the output
// index (e.g. r̃_i for σ = ⟨r̃, v⟩) may declare `Pre`, `pre(i)` and
// `post(i, val, pre, acc)`; the latency-bound products (stencil, SELL) then
// issue pre(i) together with their own loads — a plane ahead in the stencil's
// z-march — instead of after the product value is formed, which put one more
// dependent DRAM round trip on every output (`cuobjdump -sass`: the r̃ load
// sat between the last FMA and the store).  Same arithmetic, same bits.
// ---------------------------------------------------------------------------
template <class E, class = void>
struct EpiPre {
  struct P {};
  static __device__ __forceinline__ P pre(const E&, int64_t) { return P{}; }
  template <class C>
  static __device__ __forceinline__ void post(E& e, int64_t i, C val, P, double2* acc) { e(i, val, acc); }
};
template <class E>
struct EpiPre<E, std::void_t<typename E::Pre>> {
  using P = typename E::Pre;
  static __device__ __forceinline__ P pre(const E& e, int64_t i) { return e.pre(i); }
  template <class C>
  static __device__ __forceinline__ void post(E& e, int64_t i, C val, P p, double2* acc) { e.post(i, val, p, acc); }
};

// An epilogue whose early load is the product's own input at the output index
// (BsT: ⟨t, s⟩ with t = A s; CrAr: [r, A r]) says so with `pre_src()`; the
// stencil, which holds that element in a register already, then runs the
// PREX variant without the load (its active phase is L1-bound: 6 → 5 16-byte loads per point).
template <class E, class = void>
struct EpiPreSrc {
  static constexpr bool has = false;
  static const void* get(const E&) { return nullptr; }
};
template <class E>
struct EpiPreSrc<E, std::void_t<decltype(std::declval<const E&>().pre_src())>> {
  static constexpr bool has = true;
  static const void* get(const E& e) { return e.pre_src(); }
};

// An epilogue with `WANTS_X` and `post_x(i, val, pre, x_i, acc)` takes the product's own input element
// from the stencil's register (BsTm; valid where the caller guarantees input == that vector)
template <class E, class = void>
struct EpiWantsX : std::false_type {};
template <class E>
struct EpiWantsX<E, std::enable_if_t<E::WANTS_X>> : std::true_type {};

// ---------------------------------------------------------------------------
// K1 gemv_n: y_i = Σ_j A_ij x_j for local rows [0, nrows), row-major A.
// Persistent, balanced: CTA b owns rows [b·nrows/G, (b+1)·nrows/G) and walks
// them in groups of R rows.  Each thread keeps its x chunk in registers and
// reuses it across the R rows (x is read from L2 once per R rows).
// VEC: 16-byte loads (c64: 2 elements) — needs lda, n even and 16-B aligned
// pointers for c64; c128 is always 16 B per element.
// ---------------------------------------------------------------------------
template <typename T, int R, int NT, bool VEC, class Epi>
__global__ void __launch_bounds__(NT)
gemv_n_kernel(const typename CT<T>::c* __restrict__ A, int64_t lda,
              const typename CT<T>::c* __restrict__ x, int64_t n, int64_t nrows,
              Epi epi, Red red, State* st, const int* gate) {
  using C = typename CT<T>::c;
  constexpr int V = VEC ? CT<T>::V : 1;
  using LV = typename std::conditional<VEC, typename CT<T>::v, C>::type;
  constexpr int KK = Epi::K > 0 ? Epi::K : 1;
  if (pdl_gate(gate)) return;
  epi.load(st);
  __shared__ C sm[NT / 32][R];
  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);

  const int64_t rb = nrows * (int64_t)blockIdx.x / gridDim.x;
  const int64_t re = nrows * ((int64_t)blockIdx.x + 1) / gridDim.x;
  const int64_t nv = n / V;  // vector steps
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  for (int64_t g = rb; g < re; g += R) {
    const int nr = (int)min((int64_t)R, re - g);
    const LV* Ar[R];
#pragma unroll
    for (int r = 0; r < R; ++r) Ar[r] = reinterpret_cast<const LV*>(A + (g + min(r, nr - 1)) * lda);
    const LV* xv = reinterpret_cast<const LV*>(x);
    C acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = czero<C>();
#pragma unroll 2
    for (int64_t j = threadIdx.x; j < nv; j += NT) {
      C xc[V];
      unpack(__ldg(xv + j), xc);
      LV a[R];
#pragma unroll
      for (int r = 0; r < R; ++r) a[r] = ld_stream(Ar[r] + j);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        C ac[V];
        unpack(a[r], ac);
#pragma unroll
        for (int v = 0; v < V; ++v) cfma(acc[r], ac[v], xc[v]);
      }
    }
    // scalar tail (odd n with VEC)
    for (int64_t j = nv * V + threadIdx.x; j < n; j += NT) {
      C xj = x[j];
#pragma unroll
      for (int r = 0; r < R; ++r) cfma(acc[r], A[(g + min(r, nr - 1)) * lda + j], xj);
    }
    // block reduction of the R row sums (fixed order => deterministic)
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc[r].x += __shfl_xor_sync(0xffffffffu, acc[r].x, o);
        acc[r].y += __shfl_xor_sync(0xffffffffu, acc[r].y, o);
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) sm[warp][r] = acc[r];
    }
    __syncthreads();
    if (threadIdx.x < nr) {
      const int r = threadIdx.x;
      C s = sm[0][r];
#pragma unroll
      for (int w = 1; w < NT / 32; ++w) s = cadd(s, sm[w][r]);
      epi(g + r, s, dacc);
    }
    __syncthreads();
  }
  if constexpr (Epi::K > 0) finish_reduction<KK, NT, Epi>(dacc, red, st);
}

// ---------------------------------------------------------------------------
// K1' gemv_n_bulk: the same product with A streamed by the TMA bulk-copy
// engine into a STAGES-deep shared-memory ring (mbarrier tx-count pipeline),
// so the bytes in flight do not live in registers.  One CTA per SM
// (persistent), CTA b owns rows [b·nrows/G, (b+1)·nrows/G), walked in groups
// of R rows; a tile = R row segments of 4 KiB + the matching 4 KiB of x.
// Thread t owns the 16-byte column chunk t of every tile and keeps R
// accumulators; the R row sums are reduced across the CTA once per group.
// Needs n·sizeof(C) % 4096 == 0, lda·sizeof(C) % 16 == 0 and 16-B aligned A.
// ---------------------------------------------------------------------------
constexpr int BULK_TILE = 4096;  // bytes per row segment
constexpr int BULK_NT = 256;     // threads: 256 x 16 B = one 4 KiB segment

template <int R, int STAGES>
constexpr size_t bulk_smem_bytes() {
  return (size_t)STAGES * (R + 1) * BULK_TILE + 2 * STAGES * sizeof(uint64_t) + 128;
}

template <typename T, int R, int STAGES, class Epi>
__global__ void __launch_bounds__(BULK_NT, 1)
gemv_n_bulk(const typename CT<T>::c* __restrict__ A, int64_t lda,
            const typename CT<T>::c* __restrict__ x, int64_t n, int64_t nrows,
            Epi epi, Red red, State* st, const int* gate) {
  using C = typename CT<T>::c;
  using LV = typename CT<T>::v;
  constexpr int V = CT<T>::V;
  constexpr int KK = Epi::K > 0 ? Epi::K : 1;
  constexpr int TC = BULK_TILE / (int)sizeof(C);   // complex per row segment
  if (pdl_gate(gate)) return;
  epi.load(st);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* tiles = smem_raw;                                  // [STAGES][R+1][4096]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)STAGES * (R + 1) * BULK_TILE);
  uint64_t* empty = full + STAGES;
  __shared__ C red_sm[BULK_NT / 32][R];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rb = nrows * (int64_t)blockIdx.x / gridDim.x;
  const int64_t re = nrows * ((int64_t)blockIdx.x + 1) / gridDim.x;
  const int64_t ngroups = (re - rb + R - 1) / R;
  const int ntiles = (int)(n / TC);
  const int64_t tot = ngroups * ntiles;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], BULK_NT / 32); }
    fence_mbar_init();
  }
  __syncthreads();

  uint64_t pol = 0;
  auto issue = [&](int64_t t) {
    const int s = (int)(t % STAGES);
    const int64_t g = t / ntiles;
    const int ct = (int)(t % ntiles);
    const int64_t r0 = rb + g * R;
    const int nr = (int)min((int64_t)R, re - r0);
    unsigned char* stg = tiles + (size_t)s * (R + 1) * BULK_TILE;
    mbar_arrive_expect_tx(&full[s], (uint32_t)(nr + 1) * BULK_TILE);
    for (int r = 0; r < nr; ++r)
      bulk_g2s(stg + (size_t)r * BULK_TILE, A + (r0 + r) * lda + (int64_t)ct * TC, BULK_TILE, &full[s], pol);
    bulk_g2s(stg + (size_t)R * BULK_TILE, x + (int64_t)ct * TC, BULK_TILE, &full[s], pol);
  };
  if (tid == 0) {
    pol = policy_evict_first();
    for (int64_t t = 0; t < tot && t < STAGES; ++t) issue(t);
  }

  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);
  C acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = czero<C>();

  for (int64_t t = 0; t < tot; ++t) {
    const int s = (int)(t % STAGES);
    const uint32_t ph = (uint32_t)((t / STAGES) & 1);
    mbar_wait(&full[s], ph);
    const unsigned char* stg = tiles + (size_t)s * (R + 1) * BULK_TILE;
    C xc[V];
    unpack(*reinterpret_cast<const LV*>(stg + (size_t)R * BULK_TILE + tid * 16), xc);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      C ac[V];
      unpack(*reinterpret_cast<const LV*>(stg + (size_t)r * BULK_TILE + tid * 16), ac);
#pragma unroll
      for (int v = 0; v < V; ++v) cfma(acc[r], ac[v], xc[v]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (tid == 0 && t + STAGES < tot) {
      mbar_wait(&empty[s], ph);
      issue(t + STAGES);
    }
    if ((int)(t % ntiles) == ntiles - 1) {
      // end of a row group: CTA reduction of the R row sums, then epilogue
      const int64_t r0 = rb + (t / ntiles) * R;
      const int nr = (int)min((int64_t)R, re - r0);
#pragma unroll
      for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          acc[r].x += __shfl_xor_sync(0xffffffffu, acc[r].x, o);
          acc[r].y += __shfl_xor_sync(0xffffffffu, acc[r].y, o);
        }
      }
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) red_sm[warp][r] = acc[r];
      }
      __syncthreads();
      if (tid < nr) {
        C sum = red_sm[0][tid];
#pragma unroll
        for (int w = 1; w < BULK_NT / 32; ++w) sum = cadd(sum, red_sm[w][tid]);
        epi(r0 + tid, sum, dacc);
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = czero<C>();
    }
  }
  if constexpr (Epi::K > 0) finish_reduction<KK, BULK_NT, Epi>(dacc, red, st);
}

// ---------------------------------------------------------------------------
// K1'' gemv_n_split (default A·x): column strips × row blocks.  CTA (c, b)
// stages the x strip [c·W, c·W + W) in shared memory once, then each warp
// streams whole row segments of its rows (lanes 16 B apart, UR independent
// 16-byte loads in flight per lane, ~40 registers => 8 CTAs/SM, >200 KB of
// loads in flight per SM) and warp-reduces each row.  With one strip the row
// sum is final and the epilogue runs here (FUSED); otherwise the partial
// goes to part[c][i] and either gemv_h_stage2 sums the strips in order (fixed
// order => deterministic) and runs the epilogue, or (FUSED, several strips)
// the last of the row block's strip CTAs to finish — an arrival ticket per
// row block, rbt[b] — sums the strips of its rows in the same order as
// gemv_h_stage2 (bitwise the same product), runs the epilogue and puts the
// phase partials in reduction slot b: no second launch per product.
// ---------------------------------------------------------------------------
// x staging: XLoad reads the input vector; a method's input transform (e.g.
// BiCGSTAB's p = r + β(p − ωv), methods.cuh BsPIn) forms each staged element
// from other vectors instead, so that vector pass is not a launch of its own
template <typename T>
struct XLoad {
  using C = typename CT<T>::c;
  __device__ void load(const State*) {}
  __device__ C operator()(const C* x, int64_t j) const { return x[j]; }
};
template <class XIn> struct is_xload : std::false_type {};
template <typename T> struct is_xload<XLoad<T>> : std::true_type {};
// a gathered input element: the read-only-path load for the plain vector,
// else the method's input transform
template <class XIn, typename C>
__device__ __forceinline__ C xgather(const XIn& xin, const C* __restrict__ x, int64_t j) {
  if constexpr (is_xload<XIn>::value) return __ldg(x + j);
  else return xin(x, j);
}

template <typename T, int NT, int UR, bool VEC, bool FUSED, class Epi, class XIn = XLoad<T>>
__global__ void __launch_bounds__(NT)
gemv_n_split(const typename CT<T>::c* __restrict__ A, int64_t lda,
             const typename CT<T>::c* __restrict__ x, int64_t n, int64_t nrows, int W,
             typename CT<T>::c* __restrict__ part, Epi epi, Red red, State* st, const int* gate, int pin,
             unsigned* rbt, XIn xin) {
  using C = typename CT<T>::c;
  constexpr int V = VEC ? CT<T>::V : 1;
  using LV = typename std::conditional<VEC, typename CT<T>::v, C>::type;
  constexpr int KK = Epi::K > 0 ? Epi::K : 1;
  if (pdl_gate(gate)) return;
  if constexpr (FUSED) epi.load(st);
  extern __shared__ __align__(16) unsigned char xs_raw[];
  C* xs = reinterpret_cast<C*>(xs_raw);
  const int strip = blockIdx.x, nrb = gridDim.y, b = blockIdx.y;
  const int64_t c0 = (int64_t)strip * W;
  const int cw = (int)min((int64_t)W, n - c0);
  xin.load(st);
  for (int t = threadIdx.x; t < cw; t += NT) xs[t] = xin(x, c0 + t);
  __syncthreads();
  const int64_t i0 = nrows * b / nrb, i1 = nrows * (b + 1) / nrb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nvec = cw / V;
  const LV* xv = reinterpret_cast<const LV*>(xs);
  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);
  auto rows = [&](auto ld) {
  for (int64_t i = i0 + warp; i < i1; i += NT / 32) {
    const LV* a = reinterpret_cast<const LV*>(A + i * lda + c0);
    C acc = czero<C>();
    int k = lane;
    for (; k + 32 * (UR - 1) < nvec; k += 32 * UR) {
      LV av[UR];
#pragma unroll
      for (int u = 0; u < UR; ++u) av[u] = ld(a + k + 32 * u, i);
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        C ac[V], xc[V];
        unpack(av[u], ac);
        unpack(xv[k + 32 * u], xc);
#pragma unroll
        for (int v = 0; v < V; ++v) cfma(acc, ac[v], xc[v]);
      }
    }
    for (; k < nvec; k += 32) {
      C ac[V], xc[V];
      unpack(ld(a + k, i), ac);
      unpack(xv[k], xc);
#pragma unroll
      for (int v = 0; v < V; ++v) cfma(acc, ac[v], xc[v]);
    }
    if (VEC && (cw % V) && lane == 0) cfma(acc, A[i * lda + c0 + cw - 1], xs[cw - 1]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) {
      if (FUSED && gridDim.x == 1) epi(i, acc, dacc);
      else part[(int64_t)strip * nrows + i] = acc;
    }
  }
  };
  if (pin > 0) rows(make_ldpin(pin)); else rows(LdA{});
  if constexpr (FUSED) {
    if (gridDim.x > 1) {
      // strip partials of this row block: the last CTA to arrive finishes them
      __shared__ int am_last;
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        am_last = atomicAdd(rbt + b, 1u) == gridDim.x - 1;
        if (am_last) rbt[b] = 0u;   // ready for the next launch
      }
      __syncthreads();
      if (!am_last) return;
      __threadfence();
      for (int64_t i = i0 + threadIdx.x; i < i1; i += NT) {
        double2 w = make_double2(0.0, 0.0);
        for (int c = 0; c < (int)gridDim.x; ++c) {
          const C p = __ldcg(part + (int64_t)c * nrows + i);
          w.x += (double)p.x; w.y += (double)p.y;
        }
        epi(i, fromd2<C>(w), dacc);
      }
      if constexpr (Epi::K > 0) finish_reduction_at<KK, NT, Epi>(dacc, red, st, (unsigned)b, (unsigned)nrb);
    } else if constexpr (Epi::K > 0) {
      finish_reduction<KK, NT, Epi>(dacc, red, st);
    }
  }
}

// ---------------------------------------------------------------------------
// K2 stage 1: part[s][j] = Σ_{i in split s} op(A_ij) x_i, op = conj (Aᴴ) or
// identity (Aᵀ), reading row-major A once (no Aᴴ copy).  Grid (strips, S):
// CTA (c, s) owns columns [c·NT·V, (c+1)·NT·V) and rows of split s.
// x (local rows) is staged through shared memory in chunks.
// ---------------------------------------------------------------------------
template <typename T, bool CONJ, int NT, int UR, bool VEC>
__global__ void __launch_bounds__(NT)
gemv_h_stage1(const typename CT<T>::c* __restrict__ A, int64_t lda,
              const typename CT<T>::c* __restrict__ x, int64_t nrows, int64_t n,
              typename CT<T>::c* __restrict__ part, const int* gate, int pin) {
  using C = typename CT<T>::c;
  constexpr int V = VEC ? CT<T>::V : 1;
  using LV = typename std::conditional<VEC, typename CT<T>::v, C>::type;
  constexpr int CH = 512;  // rows of x per smem chunk
  if (pdl_gate(gate)) return;
  __shared__ C xs[CH];
  const int S = gridDim.y, s = blockIdx.y;
  const int64_t i0 = nrows * s / S, i1 = nrows * (s + 1) / S;
  const int64_t jv = (int64_t)blockIdx.x * NT + threadIdx.x;   // vector column index
  const int64_t nv = n / V;
  const bool active = jv < nv;
  const int64_t jc = active ? jv : 0;
  C acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = czero<C>();

  auto chunks = [&](auto ld) {
  for (int64_t c0 = i0; c0 < i1; c0 += CH) {
    const int cn = (int)min((int64_t)CH, i1 - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < cn; t += NT) xs[t] = x[c0 + t];
    __syncthreads();
    const LV* Ap = reinterpret_cast<const LV*>(A + c0 * lda) + jc;
    const int64_t ldv = lda / V;
    int t = 0;
    for (; t + UR <= cn; t += UR) {
      LV a[UR];
#pragma unroll
      for (int u = 0; u < UR; ++u) a[u] = ld(Ap + (int64_t)(t + u) * ldv, c0 + t + u);
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        C ac[V];
        unpack(a[u], ac);
        const C xi = xs[t + u];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          if (CONJ) cfmac(acc[v], ac[v], xi); else cfma(acc[v], ac[v], xi);
        }
      }
    }
    for (; t < cn; ++t) {
      C ac[V];
      unpack(ld(Ap + (int64_t)t * ldv, c0 + t), ac);
      const C xi = xs[t];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (CONJ) cfmac(acc[v], ac[v], xi); else cfma(acc[v], ac[v], xi);
      }
    }
  }
  };
  if (pin > 0) chunks(make_ldpin(pin)); else chunks(LdA{});
  if (active) {
#pragma unroll
    for (int v = 0; v < V; ++v) part[(int64_t)s * n + jv * V + v] = acc[v];
  }
  // scalar tail column (odd n with VEC): handled by strip 0, thread 0
  if (VEC && (n % V) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t j = n - 1;
    C a2 = czero<C>();
    for (int64_t i = i0; i < i1; ++i) {
      if (CONJ) cfmac(a2, A[i * lda + j], x[i]); else cfma(a2, A[i * lda + j], x[i]);
    }
    part[(int64_t)s * n + j] = a2;
  }
}

// ---------------------------------------------------------------------------
// K1c / K2D gemv_cols: the column-owner layout of K2 applied to A·x, and to
// A·x and Aᴴ·x together.  CTA (c, s) owns the column strip
// [c·NT·V, (c+1)·NT·V) — thread t the 16-byte chunk t — and the rows of split
// s, walked UR = 8 rows at a time (8 independent 16-B loads in flight per
// thread: the CTA reads 8 whole 4-KiB row segments at once, no A reuse).
//   DO_N: row partials Σ_{j∈strip} A_ij xn_j, reduced over the CTA's threads
//         (transposed warp reduction, 9 shuffle pairs per 8 rows, then the
//         warps in fixed order through double-buffered shared memory) and
//         stored to npart[c][i] — gemv_h_stage2 sums the strips in order;
//   DO_H: column partials Σ_{i∈split} op(A_ij) xh_i, op = conj (Aᴴ) or
//         identity (Aᵀ), stored to hpart[s][j] — gemv_h_stage2 sums the splits.
// With both, A·p and Aᴴ·q of one QMR iteration (they are
// independent) come out of ONE pass over A.  Needs the
// vectorised layout (16-B aligned A, lda·sizeof(C) % 16 == 0, n % V == 0).
// ---------------------------------------------------------------------------
template <typename C>
__device__ __forceinline__ void shfl_c(C& v, int o) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, o);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, o);
}

// v[0..N-1]: per-lane partials of N rows (N = 8 or 32).  Transposed warp
// reduction: at each halving step lanes with the offset bit set keep the upper
// half of their values and send the lower half (N−1 shuffle pairs in all), then
// a plain butterfly over the remaining offsets.  Afterwards lane L holds, in
// v[0], the warp sum of row L >> (5 − log2 N) (fixed order: deterministic).
template <int N, typename C>
__device__ __forceinline__ void warp_transpose_reduce(C (&v)[N], int lane) {
  static_assert(N == 8 || N == 32, "N rows");
#pragma unroll
  for (int m = N, o = 16; m > 1; m >>= 1, o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int j = 0; j < m / 2; ++j) {
      C send = up ? v[j] : v[j + m / 2];
      const C keep = up ? v[j + m / 2] : v[j];
      shfl_c(send, o);
      v[j] = cadd(keep, send);
    }
  }
#pragma unroll
  for (int o = 32 / N / 2; o >= 1; o >>= 1) {
    C t = v[0];
    shfl_c(t, o);
    v[0] = cadd(v[0], t);
  }
}

template <typename T, int NT, bool DO_N, bool DO_H, bool CONJ, int RG = 1>
__global__ void __launch_bounds__(NT)
gemv_cols(const typename CT<T>::c* __restrict__ A, int64_t lda,
          const typename CT<T>::c* __restrict__ xn, const typename CT<T>::c* __restrict__ xh,
          int64_t nrows, int64_t n, typename CT<T>::c* __restrict__ npart,
          typename CT<T>::c* __restrict__ hpart, const int* gate, int pin) {
  using C = typename CT<T>::c;
  using LV = typename CT<T>::v;
  constexpr int V = CT<T>::V;
  constexpr int UR = 8;          // rows per group of loads in flight
  constexpr int NR = UR * RG;    // rows per CTA reduction (RG groups)
  constexpr int CH = 512;        // rows of xh per shared-memory chunk (multiple of NR)
  static_assert(!(DO_H && RG != 1), "dual product: one group per reduction");
  if (pdl_gate(gate)) return;
  __shared__ C xs[DO_H ? CH : 1];
  __shared__ C red[2][NT / 32][NR];
  const int S = gridDim.y, s = blockIdx.y;
  const int64_t i0 = nrows * s / S, i1 = nrows * (s + 1) / S;
  const int64_t jv = (int64_t)blockIdx.x * NT + threadIdx.x;  // 16-byte chunk index
  const int64_t nv = n / V;
  const bool active = jv < nv;
  const int64_t jc = active ? jv : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ldv = lda / V;
  C xr[V];
#pragma unroll
  for (int v = 0; v < V; ++v) xr[v] = czero<C>();
  if (DO_N && active) unpack(*reinterpret_cast<const LV*>(xn + jv * V), xr);
  C hacc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) hacc[v] = czero<C>();
  const LV* Ab = reinterpret_cast<const LV*>(A) + jc;
  int buf = 0;
  auto chunks = [&](auto ld) {
  for (int64_t c0 = i0; c0 < i1; c0 += CH) {
    const int cn = (int)min((int64_t)CH, i1 - c0);
    if constexpr (DO_H) {
      __syncthreads();
      for (int t = threadIdx.x; t < cn; t += NT) xs[t] = xh[c0 + t];
      __syncthreads();
    }
    for (int t = 0; t < cn; t += NR) {
      const int nr = min(NR, cn - t);
      C rp[NR];
#pragma unroll
      for (int g = 0; g < RG; ++g) {
        LV a[UR];
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const int64_t row = c0 + t + min(g * UR + u, nr - 1);
          a[u] = ld(Ab + row * ldv, row);
        }
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          C ac[V];
          unpack(a[u], ac);
          C& r = rp[g * UR + u];
          r = czero<C>();
          if (DO_N && active) {
#pragma unroll
            for (int v = 0; v < V; ++v) cfma(r, ac[v], xr[v]);
          }
          if (DO_H && u < nr) {
            const C xi = xs[t + u];
#pragma unroll
            for (int v = 0; v < V; ++v) {
              if (CONJ) cfmac(hacc[v], ac[v], xi); else cfma(hacc[v], ac[v], xi);
            }
          }
        }
      }
      if constexpr (DO_N) {
        warp_transpose_reduce<NR>(rp, lane);
        constexpr int SH = NR == 32 ? 0 : 2;
        if ((lane & ((1 << SH) - 1)) == 0) red[buf][warp][lane >> SH] = rp[0];
        __syncthreads();
        if (threadIdx.x < nr) {
          C sum = red[buf][0][threadIdx.x];
#pragma unroll
          for (int w = 1; w < NT / 32; ++w) sum = cadd(sum, red[buf][w][threadIdx.x]);
          npart[(int64_t)blockIdx.x * nrows + c0 + t + threadIdx.x] = sum;
        }
        buf ^= 1;
      }
    }
  }
  };
  if (pin > 0) chunks(make_ldpin(pin)); else chunks(LdA{});
  if (DO_H && active) {
#pragma unroll
    for (int v = 0; v < V; ++v) hpart[(int64_t)s * n + jv * V + v] = hacc[v];
  }
}

// ---------------------------------------------------------------------------
// K1s gemv_sym: y = A·x (CONJ: y = conj(A)·x = Aᴴx) for complex-symmetric
// A = Aᵀ (CCG_FLAG_SYMMETRIC, one rank holding every row), reading only the
// upper triangle j ≥ i — half of A's bytes per product:
//   y_i = Σ_{j ≥ i} A_ij x_j + Σ_{j < i} A_ji x_j     (A_ij = A_ji).
// Tiles (strip c of CW = 256·V columns = 4 KiB of a row, row block I of H
// rows) of the upper triangle only (host table `tiles`, row-block major).  A
// warp takes whole 4-KiB row segments: lane l loads the 16-byte chunks
// l + 32u (u < 8) of row i — 8 independent loads — and each
// element feeds
//   N: the row dot Σ_j A_ij x_j (j ≥ i): FMAs, then a shuffle tree per row,
//      lane 0 stores npart[c][i];
//   H: the column sums Σ_i A_ij x_i (i < j): per-lane accumulators for the
//      lane's 8 chunks over the warp's rows; the 8 warps' accumulators are
//      added in warp order through shared memory once per tile -> hpart[I][j].
// No block barrier inside the row loop.  x of the strip's columns and of the
// tile's rows are staged in shared memory.  The diagonal-straddling tiles mask
// by selects and skip the chunks wholly left of the diagonal (not loaded).
// gemv_sym_stage2 sums both partial sets in a fixed order (deterministic).
// ---------------------------------------------------------------------------
constexpr int SYM_HMAX = 512;
#ifndef CCG_SYM_MINB
#define CCG_SYM_MINB 2
#endif
// XIn: input transform applied while staging x (BiCGSTAB's P / S folds,
// methods.cuh BsPIn / BsSIn; the stage-2 epilogue stores the element)
template <typename T, int NT, bool CONJ, class XIn = XLoad<T>>
__global__ void __launch_bounds__(NT, CCG_SYM_MINB)
gemv_sym(const typename CT<T>::c* __restrict__ A, int64_t lda, const typename CT<T>::c* __restrict__ x, int64_t n,
         int H, const int2* __restrict__ tiles, typename CT<T>::c* __restrict__ npart,
         typename CT<T>::c* __restrict__ hpart, const int* gate, int pin, const State* st, XIn xin) {
  using C = typename CT<T>::c;
  using LV = typename CT<T>::v;
  constexpr int V = CT<T>::V;
  constexpr int U = 8;                 // chunks per lane per row
  constexpr int CW = 32 * U * V;       // strip width in columns (4 KiB)
  constexpr int NW = NT / 32;
  static_assert(NT == 256, "gemv_sym: 8 warps");
  if (pdl_gate(gate)) return;
  __shared__ __align__(16) C xcol[CW];
  __shared__ C xrow[SYM_HMAX];
  __shared__ __align__(16) C hred[NW][CW];
  const int2 tl = tiles[blockIdx.x];
  const int c = tl.x, I = tl.y;
  const int64_t cbeg = (int64_t)c * CW, cend = min(cbeg + CW, n);
  const int64_t r0 = (int64_t)I * H, r1 = min(r0 + H, cend);
  const int rn = (int)(r1 - r0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  xin.load(st);
  for (int t = threadIdx.x; t < CW; t += NT) xcol[t] = cbeg + t < n ? xin(x, cbeg + t) : czero<C>();
  for (int t = threadIdx.x; t < rn; t += NT) xrow[t] = xin(x, r0 + t);
  __syncthreads();
  // this lane's chunks: k = lane + 32u, columns cbeg + kV .. + V − 1
  bool act[U];
#pragma unroll
  for (int u = 0; u < U; ++u) act[u] = cbeg + (int64_t)(lane + 32 * u) * V < cend;
  C hacc[U][V];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int v = 0; v < V; ++v) hacc[u][v] = czero<C>();
  const LV* Ab = reinterpret_cast<const LV*>(A + cbeg) + lane;
  const int64_t ldv = lda / V;
  const LV* xv = reinterpret_cast<const LV*>(xcol) + lane;
  auto body = [&](auto ld, auto dg) {
    constexpr bool DG = decltype(dg)::value;
    for (int t = warp; t < rn; t += NW) {   // (unroll 2 spills at 128 registers)
      const int64_t row = r0 + t;
      LV a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j0 = cbeg + (int64_t)(lane + 32 * u) * V;
        const bool need = act[u] && (!DG || j0 + V - 1 >= row);
        a[u] = need ? ld(Ab + row * ldv + 32 * u, row) : LV{};
      }
      const C xi = xrow[t];
      C acc = czero<C>();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        C ac[V], xc[V];
        unpack(a[u], ac);
        unpack(xv[32 * u], xc);
        const int64_t j0 = cbeg + (int64_t)(lane + 32 * u) * V;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          if (!DG) {
            if (CONJ) { cfmac(acc, ac[v], xc[v]); cfmac(hacc[u][v], ac[v], xi); }
            else { cfma(acc, ac[v], xc[v]); cfma(hacc[u][v], ac[v], xi); }
          } else {
            C tn = acc, th = hacc[u][v];
            if (CONJ) { cfmac(tn, ac[v], xc[v]); cfmac(th, ac[v], xi); }
            else { cfma(tn, ac[v], xc[v]); cfma(th, ac[v], xi); }
            const bool n_ok = j0 + v >= row, h_ok = j0 + v > row;
            acc.x = n_ok ? tn.x : acc.x; acc.y = n_ok ? tn.y : acc.y;
            hacc[u][v].x = h_ok ? th.x : hacc[u][v].x; hacc[u][v].y = h_ok ? th.y : hacc[u][v].y;
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {   // butterfly: every lane ends with the same sum
        C t = acc;
        shfl_c(t, o);
        acc = cadd(acc, t);
      }
      if (lane == 0) npart[(int64_t)c * n + row] = acc;
    }
  };
  const bool diag = r1 > cbeg;   // the tile reaches the diagonal: masks
  if (pin > 0) {
    if (diag) body(make_ldpin(pin), std::true_type{}); else body(make_ldpin(pin), std::false_type{});
  } else {
    if (diag) body(LdA{}, std::true_type{}); else body(LdA{}, std::false_type{});
  }
  // column sums: the warps' accumulators in warp order
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int v = 0; v < V; ++v) hred[warp][(lane + 32 * u) * V + v] = hacc[u][v];
  __syncthreads();
  for (int t = threadIdx.x; t < CW; t += NT) {
    if (cbeg + t >= n) break;
    C s = hred[0][t];
#pragma unroll
    for (int w = 1; w < NW; ++w) s = cadd(s, hred[w][t]);
    hpart[(int64_t)I * n + cbeg + t] = s;
  }
}

// bitwise equality of two complex values (their stored bit patterns)
__device__ __forceinline__ bool memcmp_c(float2 a, float2 b) {
  return __float_as_uint(a.x) == __float_as_uint(b.x) && __float_as_uint(a.y) == __float_as_uint(b.y);
}
__device__ __forceinline__ bool memcmp_c(double2 a, double2 b) {
  return __double_as_longlong(a.x) == __double_as_longlong(b.x) &&
         __double_as_longlong(a.y) == __double_as_longlong(b.y);
}

// Exact symmetry test A = Aᵀ (ccg_set_matvec_dense without CCG_FLAG_SYMMETRIC,
// one rank): 32×32 tile pairs (I ≤ J) of the upper triangle, the lower tile
// transposed through shared memory, the 16-byte patterns compared bitwise.
// The first mismatch sets *bad and every CTA stops at its next tile, so a
// general matrix costs a few tiles; a symmetric one one read of A.
template <typename T>
__global__ void __launch_bounds__(256)
sym_check(const typename CT<T>::c* __restrict__ A, int64_t lda, int64_t n, int* bad) {
  using C = typename CT<T>::c;
  __shared__ C lo[32][33];
  __shared__ int stop;
  const int64_t NTL = (n + 31) / 32;
  const int64_t pairs = NTL * (NTL + 1) / 2;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 × 8
  for (int64_t p = blockIdx.x; p < pairs; p += gridDim.x) {
    if (threadIdx.x == 0) stop = *(volatile int*)bad;
    __syncthreads();
    if (stop) return;
    // p -> (I, J), I ≤ J: row-major enumeration of the upper triangle of tiles
    int64_t I = (int64_t)((2 * NTL + 1 - sqrt((double)(2 * NTL + 1) * (2 * NTL + 1) - 8.0 * (double)p)) / 2);
    while (I > 0 && I * NTL - I * (I - 1) / 2 > p) --I;
    while ((I + 1) * NTL - (I + 1) * I / 2 <= p) ++I;
    const int64_t J = I + (p - (I * NTL - I * (I - 1) / 2));
    bool ok = true;
    for (int r = ty; r < 32; r += 8) {   // lower tile (J, I) -> shared, transposed on read
      const int64_t i = J * 32 + r, j = I * 32 + tx;
      if (i < n && j < n) lo[r][tx] = A[i * lda + j];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {   // upper tile (I, J): A[I*32+r][J*32+tx] vs A[J*32+tx][I*32+r]
      const int64_t i = I * 32 + r, j = J * 32 + tx;
      if (i < n && j < n) {
        const C a = A[i * lda + j], b = lo[tx][r];
        ok &= memcmp_c(a, b);
      }
    }
    // one atomic per CTA (a per-thread atomic on one address serialised
    // ~300 k of them on a general matrix: 220 µs instead of a few)
    if (__syncthreads_or(!ok) && threadIdx.x == 0) atomicExch(bad, 1);
  }
}

// K1s' gemv_sym_dual: A·p and Aᴴ·q of one QMR / BiCG iteration (independent,
// SURVEY §8(a) a7; §8(f) NEXT-1) from ONE pass over the upper triangle of a
// complex-symmetric A — half of the full dual pass's bytes, the same as one
// gemv_sym.  Each loaded element feeds four sums:
//   (A p)_i:  N Σ_{j≥i} A_ij p_j,        H Σ_{i<j} A_ij p_i      -> np1 / hp1
//   (Aᴴq)_i:  N Σ_{j≥i} conj(A_ij) q_j,  H Σ_{i<j} conj(A_ij) q_i -> np2 / hp2
// Same layout as gemv_sym with 4 chunks per lane (2-KiB strips: CW = 128·V)
// so the two sets of column accumulators fit the register budget.
template <typename T, int NT>
__global__ void __launch_bounds__(NT, 2)
gemv_sym_dual(const typename CT<T>::c* __restrict__ A, int64_t lda, const typename CT<T>::c* __restrict__ p,
              const typename CT<T>::c* __restrict__ q, int64_t n, int H, const int2* __restrict__ tiles,
              typename CT<T>::c* __restrict__ np1, typename CT<T>::c* __restrict__ hp1,
              typename CT<T>::c* __restrict__ np2, typename CT<T>::c* __restrict__ hp2, const int* gate) {
  using C = typename CT<T>::c;
  using LV = typename CT<T>::v;
  constexpr int V = CT<T>::V;
  constexpr int U = 4;
  constexpr int CW = 32 * U * V;
  constexpr int NW = NT / 32;
  static_assert(NT == 256, "gemv_sym_dual: 8 warps");
  if (pdl_gate(gate)) return;
  __shared__ __align__(16) C pcol[CW];
  __shared__ __align__(16) C qcol[CW];
  __shared__ C prow[SYM_HMAX];
  __shared__ C qrow[SYM_HMAX];
  __shared__ __align__(16) C hred[NW][CW];
  const int2 tl = tiles[blockIdx.x];
  const int c = tl.x, I = tl.y;
  const int64_t cbeg = (int64_t)c * CW, cend = min(cbeg + CW, n);
  const int64_t r0 = (int64_t)I * H, r1 = min(r0 + H, cend);
  const int rn = (int)(r1 - r0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < CW; t += NT) {
    pcol[t] = cbeg + t < n ? p[cbeg + t] : czero<C>();
    qcol[t] = cbeg + t < n ? q[cbeg + t] : czero<C>();
  }
  for (int t = threadIdx.x; t < rn; t += NT) { prow[t] = p[r0 + t]; qrow[t] = q[r0 + t]; }
  __syncthreads();
  bool act[U];
#pragma unroll
  for (int u = 0; u < U; ++u) act[u] = cbeg + (int64_t)(lane + 32 * u) * V < cend;
  C h1[U][V], h2[U][V];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int v = 0; v < V; ++v) { h1[u][v] = czero<C>(); h2[u][v] = czero<C>(); }
  const LV* Ab = reinterpret_cast<const LV*>(A + cbeg) + lane;
  const int64_t ldv = lda / V;
  const LV* pv = reinterpret_cast<const LV*>(pcol) + lane;
  const LV* qv = reinterpret_cast<const LV*>(qcol) + lane;
  // two rows per step (t, t + 1): 8 loads in flight per lane, and the row sums
  // of the pair share one transposed shuffle level (lanes 0-15 keep row t,
  // lanes 16-31 row t + 1), then a 4-level butterfly inside each half
  auto body = [&](auto dg) {
    constexpr bool DG = decltype(dg)::value;
    for (int t = 2 * warp; t < rn; t += 2 * NW) {
      LV a[2][U];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int tr = min(t + r, rn - 1);
        const int64_t row = r0 + tr;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t j0 = cbeg + (int64_t)(lane + 32 * u) * V;
          const bool need = act[u] && (t + r < rn) && (!DG || j0 + V - 1 >= row);
          a[r][u] = need ? ld_stream(Ab + row * ldv + 32 * u) : LV{};
        }
      }
      C n1[2], n2[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int tr = min(t + r, rn - 1);
        const int64_t row = r0 + tr;
        const C pi = prow[tr], qi = qrow[tr];
        const bool live = t + r < rn;
        n1[r] = czero<C>(); n2[r] = czero<C>();
#pragma unroll
        for (int u = 0; u < U; ++u) {
          C ac[V], pc[V], qc[V];
          unpack(a[r][u], ac);
          unpack(pv[32 * u], pc);
          unpack(qv[32 * u], qc);
          const int64_t j0 = cbeg + (int64_t)(lane + 32 * u) * V;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            C t1 = n1[r], t2 = n2[r], t3 = h1[u][v], t4 = h2[u][v];
            cfma(t1, ac[v], pc[v]);
            cfmac(t2, ac[v], qc[v]);
            cfma(t3, ac[v], pi);
            cfmac(t4, ac[v], qi);
            const bool n_ok = !DG || j0 + v >= row, h_ok = live && (!DG || j0 + v > row);
            n1[r].x = n_ok ? t1.x : n1[r].x; n1[r].y = n_ok ? t1.y : n1[r].y;
            n2[r].x = n_ok ? t2.x : n2[r].x; n2[r].y = n_ok ? t2.y : n2[r].y;
            h1[u][v].x = h_ok ? t3.x : h1[u][v].x; h1[u][v].y = h_ok ? t3.y : h1[u][v].y;
            h2[u][v].x = h_ok ? t4.x : h2[u][v].x; h2[u][v].y = h_ok ? t4.y : h2[u][v].y;
          }
        }
      }
      const bool up = lane & 16;
      C s1 = up ? n1[0] : n1[1], s2 = up ? n2[0] : n2[1];
      C k1 = up ? n1[1] : n1[0], k2 = up ? n2[1] : n2[0];
      shfl_c(s1, 16);
      shfl_c(s2, 16);
      k1 = up ? cadd(s1, k1) : cadd(k1, s1);   // lane l and l ^ 16 add in the same order
      k2 = up ? cadd(s2, k2) : cadd(k2, s2);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        C t1 = k1, t2 = k2;
        shfl_c(t1, o);
        shfl_c(t2, o);
        k1 = cadd(k1, t1);
        k2 = cadd(k2, t2);
      }
      const int r = up ? 1 : 0;
      if ((lane & 15) == 0 && t + r < rn) {
        np1[(int64_t)c * n + r0 + t + r] = k1;
        np2[(int64_t)c * n + r0 + t + r] = k2;
      }
    }
  };
  if (r1 > cbeg) body(std::true_type{}); else body(std::false_type{});
  // column sums of both products, warps in order, through the same buffer
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int v = 0; v < V; ++v) hred[warp][(lane + 32 * u) * V + v] = h1[u][v];
  __syncthreads();
  for (int t = threadIdx.x; t < CW; t += NT) {
    if (cbeg + t >= n) break;
    C s = hred[0][t];
#pragma unroll
    for (int w = 1; w < NW; ++w) s = cadd(s, hred[w][t]);
    hp1[(int64_t)I * n + cbeg + t] = s;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int v = 0; v < V; ++v) hred[warp][(lane + 32 * u) * V + v] = h2[u][v];
  __syncthreads();
  for (int t = threadIdx.x; t < CW; t += NT) {
    if (cbeg + t >= n) break;
    C s = hred[0][t];
#pragma unroll
    for (int w = 1; w < NW; ++w) s = cadd(s, hred[w][t]);
    hp2[(int64_t)I * n + cbeg + t] = s;
  }
}

// K2D' gemv_dual_rows: A·p and Aᴴ·q of one QMR / BiCG iteration from ONE pass
// over a GENERAL A, in gemv_sym's warp-per-row layout:
// tile = (strip c of CW = 256·V columns, row block I of H rows); a warp takes
// whole 4-KiB row segments (8 independent 16-B loads per lane), forms the row
// dot with p (shuffle tree, lane 0 stores np[c][i]) and keeps per-lane column
// accumulators Σ_i conj(A_ij) q_i added over the tile's warps once (hp[I][j]).
// No barrier in the row loop (the column-owner dual, gemv_cols<DO_N, DO_H>,
// reduces its row sums across warps every 8 rows).  gemv_h_stage2 sums np over
// the strips and hp over the row blocks, each in a fixed order.
template <typename T, int NT>
__global__ void __launch_bounds__(NT, 2)
gemv_dual_rows(const typename CT<T>::c* __restrict__ A, int64_t lda, const typename CT<T>::c* __restrict__ p,
               const typename CT<T>::c* __restrict__ q, int64_t nrows, int64_t n, int H, int nstrips,
               typename CT<T>::c* __restrict__ np, typename CT<T>::c* __restrict__ hp, const int* gate) {
  using C = typename CT<T>::c;
  using LV = typename CT<T>::v;
  constexpr int V = CT<T>::V;
  constexpr int U = 8;
  constexpr int CW = 32 * U * V;
  constexpr int NW = NT / 32;
  static_assert(NT == 256, "gemv_dual_rows: 8 warps");
  if (pdl_gate(gate)) return;
  __shared__ __align__(16) C pcol[CW];
  __shared__ C qrow[SYM_HMAX];
  __shared__ __align__(16) C hred[NW][CW];
  const int c = (int)(blockIdx.x % nstrips), I = (int)(blockIdx.x / nstrips);   // row-block major
  const int64_t cbeg = (int64_t)c * CW, cend = min(cbeg + CW, n);
  const int64_t r0 = (int64_t)I * H, r1 = min(r0 + H, nrows);
  const int rn = (int)(r1 - r0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < CW; t += NT) pcol[t] = cbeg + t < n ? p[cbeg + t] : czero<C>();
  for (int t = threadIdx.x; t < rn; t += NT) qrow[t] = q[r0 + t];
  __syncthreads();
  bool act[U];
#pragma unroll
  for (int u = 0; u < U; ++u) act[u] = cbeg + (int64_t)(lane + 32 * u) * V < cend;
  C hacc[U][V];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int v = 0; v < V; ++v) hacc[u][v] = czero<C>();
  const LV* Ab = reinterpret_cast<const LV*>(A + cbeg) + lane;
  const int64_t ldv = lda / V;
  const LV* pv = reinterpret_cast<const LV*>(pcol) + lane;
  for (int t = warp; t < rn; t += NW) {
    const int64_t row = r0 + t;
    LV a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = act[u] ? ld_stream(Ab + row * ldv + 32 * u) : LV{};
    const C qi = qrow[t];
    C acc = czero<C>();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      C ac[V], pc[V];
      unpack(a[u], ac);
      unpack(pv[32 * u], pc);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        cfma(acc, ac[v], pc[v]);
        cfmac(hacc[u][v], ac[v], qi);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      C tt = acc;
      shfl_c(tt, o);
      acc = cadd(acc, tt);
    }
    if (lane == 0) np[(int64_t)c * nrows + row] = acc;
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int v = 0; v < V; ++v) hred[warp][(lane + 32 * u) * V + v] = hacc[u][v];
  __syncthreads();
  for (int t = threadIdx.x; t < CW; t += NT) {
    if (cbeg + t >= n) break;
    C sum = hred[0][t];
#pragma unroll
    for (int w = 1; w < NW; ++w) sum = cadd(sum, hred[w][t]);
    hp[(int64_t)I * n + cbeg + t] = sum;
  }
}

// y_i = Σ_{c ≥ c(i)} npart[c][i] + Σ_{I < nb(c(i))} hpart[I][i] (fp64), then
// the epilogue; c(i) = i / CW, nb(c) = the row blocks of strip c.  A CTA takes
// 32 consecutive outputs (one strip: CW is a multiple of 32), lane = output;
// warp w sums the partials p ≡ w (mod NT/32) of the list [npart strips ...,
// hpart blocks ...] in order, then warp 0 adds the warp sums in warp order —
// a fixed order (deterministic) with NT/32 independent load streams per
// output (one thread per output walking ~n/H partials was latency-bound).
template <typename T, int NT, class Epi>
__global__ void __launch_bounds__(NT)
gemv_sym_stage2(const typename CT<T>::c* __restrict__ npart, const typename CT<T>::c* __restrict__ hpart, int64_t n,
                int H, int CW, int nstrips, Epi epi, Red red, State* st, const int* gate) {
  using C = typename CT<T>::c;
  constexpr int KK = Epi::K > 0 ? Epi::K : 1;
  constexpr int NW = NT / 32;
  if (pdl_gate(gate)) return;
  epi.load(st);
  __shared__ double2 sh[NW][32];
  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = (int64_t)blockIdx.x * 32; base < n; base += (int64_t)gridDim.x * 32) {
    const int64_t i = base + lane;
    const bool valid = i < n;
    const int ci = (int)(base / CW);
    const int nN = nstrips - ci;
    const int64_t cend = min((int64_t)(ci + 1) * CW, n);
    const int P = nN + (int)((cend + H - 1) / H);
    double2 w = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int p = warp; p < P; p += NW) {
      const C* src = p < nN ? npart + (int64_t)(ci + p) * n : hpart + (int64_t)(p - nN) * n;
      if (valid) {
        const C v = __ldcs(src + i);
        w.x += (double)v.x; w.y += (double)v.y;
      }
    }
    sh[warp][lane] = w;
    __syncthreads();
    if (warp == 0) {
      double2 y = sh[0][lane];
#pragma unroll
      for (int k = 1; k < NW; ++k) { y.x += sh[k][lane].x; y.y += sh[k][lane].y; }
      if (valid) epi(i, fromd2<C>(y), dacc);
    }
    __syncthreads();
  }
  if constexpr (Epi::K > 0) finish_reduction<KK, NT, Epi>(dacc, red, st);
}

// w_j = Σ_s part[s][off + j] (fp64) with NT/32 load streams per output: a CTA
// takes 32 consecutive outputs (lane = output), warp w sums the partials
// s ≡ w (mod NT/32) in order, warp 0 adds the warp sums in warp order — a fixed
// order; for the many-partial sums of the warp-per-row dual (64 strips / row
// blocks at config 3) where one thread per output walking them was
// latency-bound (18 µs per launch)
template <typename T, int NT, class Epi>
__global__ void __launch_bounds__(NT)
part_sum_stage2(const typename CT<T>::c* __restrict__ part, int S, int64_t n, int64_t nout, Epi epi, Red red,
                State* st, const int* gate) {
  using C = typename CT<T>::c;
  constexpr int KK = Epi::K > 0 ? Epi::K : 1;
  constexpr int NW = NT / 32;
  if (pdl_gate(gate)) return;
  epi.load(st);
  __shared__ double2 sh[NW][32];
  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = (int64_t)blockIdx.x * 32; base < nout; base += (int64_t)gridDim.x * 32) {
    const int64_t j = base + lane;
    const bool valid = j < nout;
    double2 w = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int sidx = warp; sidx < S; sidx += NW) {
      if (valid) {
        const C v = __ldcs(part + (int64_t)sidx * n + j);
        w.x += (double)v.x; w.y += (double)v.y;
      }
    }
    sh[warp][lane] = w;
    __syncthreads();
    if (warp == 0) {
      double2 y = sh[0][lane];
#pragma unroll
      for (int k = 1; k < NW; ++k) { y.x += sh[k][lane].x; y.y += sh[k][lane].y; }
      if (valid) epi(j, fromd2<C>(y), dacc);
    }
    __syncthreads();
  }
  if constexpr (Epi::K > 0) finish_reduction<KK, NT, Epi>(dacc, red, st);
}

// K2 stage 2: w_j = Σ_s part[s][off + j] in split order, then epilogue.
template <typename T, int NT, class Epi>
__global__ void __launch_bounds__(NT)
gemv_h_stage2(const typename CT<T>::c* __restrict__ part, int S, int64_t n, int64_t off,
              int64_t nout, Epi epi, Red red, State* st, const int* gate) {
  using C = typename CT<T>::c;
  constexpr int KK = Epi::K > 0 ? Epi::K : 1;
  if (pdl_gate(gate)) return;
  epi.load(st);
  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);
  for (int64_t j = (int64_t)blockIdx.x * NT + threadIdx.x; j < nout; j += (int64_t)gridDim.x * NT) {
    double2 w = make_double2(0.0, 0.0);
    for (int s = 0; s < S; ++s) {
      C p = __ldcs(part + (int64_t)s * n + off + j);
      w.x += (double)p.x; w.y += (double)p.y;
    }
    epi(j, fromd2<C>(w), dacc);
  }
  if constexpr (Epi::K > 0) finish_reduction<KK, NT, Epi>(dacc, red, st);
}

// ---------------------------------------------------------------------------
// K3 CSR SpMV, LPR lanes per row (LPR = 4 or 8 for ~7 nnz/row stencils,
// 32 = warp-per-row).  Column indices are GLOBAL; x is a full-length buffer
// (own slice + halos filled).  CONJ: y = conj(A·conj(x)) (= Aᴴx for
// complex-symmetric A).
// ---------------------------------------------------------------------------
template <typename T, int LPR, int NT, bool CONJ, class Epi>
__global__ void __launch_bounds__(NT)
spmv_csr_kernel(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                const typename CT<T>::c* __restrict__ vals, const typename CT<T>::c* __restrict__ x,
                int64_t nrows, Epi epi, Red red, State* st, const int* gate) {
  using C = typename CT<T>::c;
  constexpr int KK = Epi::K > 0 ? Epi::K : 1;
  if (pdl_gate(gate)) return;
  epi.load(st);
  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);
  const int sub = threadIdx.x % LPR;
  const int64_t rows_per_iter = (int64_t)gridDim.x * (NT / LPR);
  for (int64_t i = (int64_t)blockIdx.x * (NT / LPR) + threadIdx.x / LPR; i < nrows; i += rows_per_iter) {
    const int k0 = __ldg(rowptr + i), k1 = __ldg(rowptr + i + 1);
    C acc = czero<C>();
    for (int k = k0 + sub; k < k1; k += LPR) {
      const C a = __ldcs(vals + k);
      C xv = __ldg(x + __ldcs(colind + k));
      if (CONJ) xv = cconj(xv);
      cfma(acc, a, xv);
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o, LPR);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o, LPR);
    }
    if (sub == 0) epi(i, CONJ ? cconj(acc) : acc, dacc);
  }
  if constexpr (Epi::K > 0) finish_reduction<KK, NT, Epi>(dacc, red, st);
}

// ---------------------------------------------------------------------------
// K3' CSR-stream SpMV (default): the rows are cut on the host into blocks of
// ≤ NT rows and ≤ NNZ_MAX nonzeros (a row longer than NNZ_MAX is a block of
// its own).  A CTA streams its block's vals/colind coalesced, 8 independent
// (val, col) pairs then 8 independent x gathers per thread, writes the
// products to shared memory, and thread t sums row t's products in CSR order
// (deterministic).  All loads of a block are in flight at once instead of one
// dependent rowptr → colind → x chain per row.
// ---------------------------------------------------------------------------
template <typename T, int NT, int NNZ_MAX, bool CONJ, class Epi>
__global__ void __launch_bounds__(NT)
spmv_stream_kernel(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                   const typename CT<T>::c* __restrict__ vals, const typename CT<T>::c* __restrict__ x,
                   const int32_t* __restrict__ blocks, int nblocks, Epi epi, Red red, State* st,
                   const int* gate) {
  using C = typename CT<T>::c;
  constexpr int KK = Epi::K > 0 ? Epi::K : 1;
  constexpr int U = 8;
  if (pdl_gate(gate)) return;
  epi.load(st);
  __shared__ C prod[NNZ_MAX];
  __shared__ int32_t rp[NT + 1];
  __shared__ double2 lsum[NT / 32];
  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);
  const int t = threadIdx.x;
  for (int b = blockIdx.x; b < nblocks; b += gridDim.x) {
    const int r0 = __ldg(blocks + b), r1 = __ldg(blocks + b + 1);
    const int nr = r1 - r0;
    const int k0 = __ldg(rowptr + r0), k1 = __ldg(rowptr + r1);
    if (k1 - k0 > NNZ_MAX) {
      // one long row: strided partial sums, fixed-order CTA reduction
      C acc = czero<C>();
      for (int k = k0 + t; k < k1; k += NT) {
        C xv = __ldg(x + __ldcs(colind + k));
        if (CONJ) xv = cconj(xv);
        cfma(acc, __ldcs(vals + k), xv);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if ((t & 31) == 0) lsum[t >> 5] = make_double2((double)acc.x, (double)acc.y);
      __syncthreads();
      if (t == 0) {
        C s = czero<C>();
        for (int w = 0; w < NT / 32; ++w) { s.x += lsum[w].x; s.y += lsum[w].y; }
        epi(r0, CONJ ? cconj(s) : s, dacc);
      }
      __syncthreads();
      continue;
    }
    const int nk = k1 - k0;
    for (int j = t; j <= nr; j += NT) rp[j] = __ldg(rowptr + r0 + j) - k0;
    for (int kb = t; kb < nk; kb += NT * U) {
      int col[U];
      C v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = kb + u * NT;
        col[u] = k < nk ? __ldcs(colind + k0 + k) : 0;
        v[u] = k < nk ? __ldcs(vals + k0 + k) : czero<C>();
      }
      C xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(x + col[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = kb + u * NT;
        if (k < nk) {
          C xx = CONJ ? cconj(xv[u]) : xv[u];
          C p = czero<C>();
          cfma(p, v[u], xx);
          prod[k] = p;
        }
      }
    }
    __syncthreads();
    if (t < nr) {
      C s = czero<C>();
      for (int k = rp[t]; k < rp[t + 1]; ++k) s = cadd(s, prod[k]);
      epi(r0 + t, CONJ ? cconj(s) : s, dacc);
    }
    __syncthreads();
  }
  if constexpr (Epi::K > 0) finish_reduction<KK, NT, Epi>(dacc, red, st);
}

// ---------------------------------------------------------------------------
// K3'' SELL-32 SpMV (default when padding is small, e.g. the 7-point stencil):
// the library copies the borrowed CSR once into slices of 32 consecutive rows
// stored column-major (entry j of row 32s+l at off_s + 32j + l, padding
// col = -1), so a warp reads 512 B of values + 128 B of columns per step,
// fully coalesced, one row per lane, no shared memory and no barriers.  The
// row sum runs in CSR column order (same order as the CSR kernels).
// ---------------------------------------------------------------------------
// one SELL row of exactly W stored entries: all W column indices, then all W
// values and x gathers are issued before any arithmetic (padding: col = −1,
// gather clamped to index 0 and its product skipped), then the products are
// accumulated by FMA in CSR column order
template <int W, bool CONJ, typename C, class XIn>
__device__ __forceinline__ C sell_row(const int32_t* __restrict__ scol, const C* __restrict__ sval,
                                      const C* __restrict__ x, int64_t base, const XIn& xin) {
  int col[W];
#pragma unroll
  for (int u = 0; u < W; ++u) col[u] = __ldcs(scol + base + 32 * (int64_t)u);
  C v[W], xv[W];
#pragma unroll
  for (int u = 0; u < W; ++u) {
    v[u] = __ldcs(sval + base + 32 * (int64_t)u);
    xv[u] = xgather(xin, x, max(col[u], 0));
  }
  C acc = czero<C>();
#pragma unroll
  for (int u = 0; u < W; ++u) {
    C a2 = acc;
    cfma(a2, v[u], CONJ ? cconj(xv[u]) : xv[u]);   // acc += v·x as 4 FMAs
    acc.x = col[u] >= 0 ? a2.x : acc.x;   // select, not a branch: the loads stay batched
    acc.y = col[u] >= 0 ? a2.y : acc.y;
  }
  return acc;
}

// Load schedule, chosen per dtype by measurement (tools/sweep_sell.py):
// ONE = false — two rows per step for width-7 slices, ptxas' default register
// budget (it interleaves the loads with the FMAs: ~2-3 loads in flight);
// ONE = true — one row per step with "≥ 3 CTAs/SM" in the launch bounds, under
// which ptxas issues all 14 loads of a row before its arithmetic (78-94
// registers): c128 SpMV 64.6 → 57.9 µs at config 5 (cold ncu), the default.
// XIn: input transform of the gathered x (see stencil7_kernel); CONJ = false only
template <typename T, int NT, bool CONJ, bool ONE, class Epi, class XIn = XLoad<T>>
__global__ void __launch_bounds__(NT, ONE ? 3 : 0)
spmv_sell_kernel(const int64_t* __restrict__ soff, const int32_t* __restrict__ swidth,
                 const int32_t* __restrict__ scol, const typename CT<T>::c* __restrict__ sval,
                 const typename CT<T>::c* __restrict__ x, int64_t nrows, Epi epi, Red red, State* st,
                 const int* gate, XIn xin) {
  using C = typename CT<T>::c;
  constexpr int KK = Epi::K > 0 ? Epi::K : 1;
  constexpr int U = 8;
  if (pdl_gate(gate)) return;
  epi.load(st);
  xin.load(st);
  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);
  const int64_t nwarps_rows = ((nrows + 31) / 32) * 32;
  const int64_t stride = (int64_t)gridDim.x * NT;
  int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x;
  // two rows per step (i, i + stride) when their slices share the common
  // stencil width 7: twice the loads in flight per thread
  using EP = EpiPre<Epi>;
  for (; !ONE && i + stride < nwarps_rows; i += 2 * stride) {
    const int64_t s1 = i >> 5, s2 = (i + stride) >> 5;
    const int lane = (int)(i & 31);
    const int w1 = __ldg(swidth + s1), w2 = __ldg(swidth + s2);
    if (w1 != 7 || w2 != 7) break;      // warp-uniform; the generic loop below finishes
    typename EP::P p1{}, p2{};
    if (i < nrows) p1 = EP::pre(epi, i);
    if (i + stride < nrows) p2 = EP::pre(epi, i + stride);
    const int64_t b1 = __ldg(soff + s1) + lane, b2 = __ldg(soff + s2) + lane;
    int c1[7], c2[7];
#pragma unroll
    for (int u = 0; u < 7; ++u) { c1[u] = __ldcs(scol + b1 + 32 * u); c2[u] = __ldcs(scol + b2 + 32 * u); }
    C v1[7], v2[7], x1[7], x2[7];
#pragma unroll
    for (int u = 0; u < 7; ++u) {
      v1[u] = __ldcs(sval + b1 + 32 * u); x1[u] = xgather(xin, x, max(c1[u], 0));
      v2[u] = __ldcs(sval + b2 + 32 * u); x2[u] = xgather(xin, x, max(c2[u], 0));
    }
    C a1 = czero<C>(), a2 = czero<C>();
#pragma unroll
    for (int u = 0; u < 7; ++u) {
      C t1 = a1, t2 = a2;
      cfma(t1, v1[u], CONJ ? cconj(x1[u]) : x1[u]);
      cfma(t2, v2[u], CONJ ? cconj(x2[u]) : x2[u]);
      a1.x = c1[u] >= 0 ? t1.x : a1.x; a1.y = c1[u] >= 0 ? t1.y : a1.y;
      a2.x = c2[u] >= 0 ? t2.x : a2.x; a2.y = c2[u] >= 0 ? t2.y : a2.y;
    }
    if (i < nrows) EP::post(epi, i, CONJ ? cconj(a1) : a1, p1, dacc);
    if (i + stride < nrows) EP::post(epi, i + stride, CONJ ? cconj(a2) : a2, p2, dacc);
  }
  for (; i < nwarps_rows; i += stride) {
    const int64_t s = i >> 5;
    const int lane = (int)(i & 31);
    typename EP::P pr{};
    if (i < nrows) pr = EP::pre(epi, i);
    const int w = __ldg(swidth + s);
    const int64_t base = __ldg(soff + s) + lane;
    C acc;
    switch (w) {   // warp-uniform: the whole slice shares its width
      case 0: acc = czero<C>(); break;
      case 1: acc = sell_row<1, CONJ>(scol, sval, x, base, xin); break;
      case 2: acc = sell_row<2, CONJ>(scol, sval, x, base, xin); break;
      case 3: acc = sell_row<3, CONJ>(scol, sval, x, base, xin); break;
      case 4: acc = sell_row<4, CONJ>(scol, sval, x, base, xin); break;
      case 5: acc = sell_row<5, CONJ>(scol, sval, x, base, xin); break;
      case 6: acc = sell_row<6, CONJ>(scol, sval, x, base, xin); break;
      case 7: acc = sell_row<7, CONJ>(scol, sval, x, base, xin); break;
      case 8: acc = sell_row<8, CONJ>(scol, sval, x, base, xin); break;
      default: {
        acc = czero<C>();
        for (int j0 = 0; j0 < w; j0 += U) {
          int col[U];
          C v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = j0 + u;
            col[u] = j < w ? __ldcs(scol + base + 32 * (int64_t)j) : -1;
            v[u] = j < w ? __ldcs(sval + base + 32 * (int64_t)j) : czero<C>();
          }
          C xv[U];
#pragma unroll
          for (int u = 0; u < U; ++u) xv[u] = col[u] >= 0 ? xgather(xin, x, col[u]) : czero<C>();
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (col[u] >= 0) {
              C p = czero<C>();
              cfma(p, v[u], CONJ ? cconj(xv[u]) : xv[u]);
              acc = cadd(acc, p);
            }
          }
        }
      }
    }
    if (i < nrows) EP::post(epi, i, CONJ ? cconj(acc) : acc, pr, dacc);
  }
  if constexpr (Epi::K > 0) finish_reduction<KK, NT, Epi>(dacc, red, st);
}

// CSR -> SELL-32 scatter (one thread per row), run once at ccg_set_matvec_csr
template <typename C>
__global__ void csr_to_sell(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                            const C* __restrict__ vals, const int64_t* __restrict__ soff,
                            const int32_t* __restrict__ swidth, int64_t nrows, int32_t* scol, C* sval) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ((nrows + 31) / 32) * 32) return;
  const int64_t s = i >> 5;
  const int lane = (int)(i & 31);
  const int w = swidth[s];
  const int64_t base = soff[s] + lane;
  const int k0 = i < nrows ? rowptr[i] : 0, k1 = i < nrows ? rowptr[i + 1] : 0;
  for (int j = 0; j < w; ++j) {
    const int k = k0 + j;
    C z; z.x = 0; z.y = 0;
    scol[base + 32 * (int64_t)j] = k < k1 ? colind[k] : -1;
    sval[base + 32 * (int64_t)j] = k < k1 ? vals[k] : z;
  }
}

// ---------------------------------------------------------------------------
// K3s matrix-free 7-point stencil (the paper's "own
// sparse matrix scheme" in matvec, P:95 [§5]): on an nx × ny × nz lattice
// (x fastest) with Dirichlet boundaries,
//   (A u)_p = d·u_p + ox·(u_{p±x̂}) + oy·(u_{p±ŷ}) + oz·(u_{p±ẑ}),
// neighbours outside the lattice = 0 (config 5: d = 6 − k²(1 + i/2),
// o = −1, BJ:11).  The rank owns planes [z0, z0 + nzl); x is a full-length
// buffer at global indices whose halo planes z0 − 1 and z0 + nzl are filled.
// No matrix is stored: per point one x read (L1/L2 serve the 6 neighbour
// reads; the z neighbours rotate through registers as a thread marches zc
// planes) and one y write, i.e. 2·n·s bytes instead of CSR's nnz·(s + 4).
// Terms are accumulated by FMA (acc += coef·v, 4 FMAs) in ascending column
// order — the same arithmetic as the SELL CSR kernel on the equivalent
// matrix, so the two operators give bitwise-identical products.
// Block: 256 threads = 32 (x) × 8 (y); grid (⌈nx/32⌉, ⌈ny/8⌉, ⌈nzl/zc⌉).
// ---------------------------------------------------------------------------
// Boundary handling without per-term selects (round 2; the select version was
// issue-bound: 129 SASS instructions per point with the BsT epilogue, 24 FSEL
// + 10 CS2R + ~12 predicate ops of them).  A missing x/y neighbour is handled
// once per thread, outside the z loop: its load offset is clamped to 0 (the
// thread re-reads its own point — always in bounds, and finite whenever the
// point itself is) and its coefficient is a per-thread register set to 0, so
// the loop body is 5 unconditional loads and 7 unconditional complex FMAs.
// fma(0, v, acc) leaves acc bitwise unchanged for finite v unless acc is −0,
// and acc (started at +0) can only be −0 after an underflow to −0: the product
// stays bitwise equal to the CSR one except for the sign of such a zero
// (DESIGN §4.3).  z: the plane below the lattice is a zero value; the plane
// above is a predicated load (uniform per CTA).
// REALO: ox, oy, oz have exactly zero imaginary parts (the Laplacian of
// config 5): the two FMAs per term that multiply by it are skipped (same
// caveat: they could only flip the sign of a zero component).
template <bool REALO, typename C>
__device__ __forceinline__ void st_fma(C& acc, C coef, C v) {
  if constexpr (REALO) {
    acc.x = fma(coef.x, v.x, acc.x);
    acc.y = fma(coef.x, v.y, acc.y);
  } else {
    cfma(acc, coef, v);
  }
}

// XIn: input transform (as in gemv_n_split) — each lattice value is formed as
// xin(x, j) from other vectors (BiCGSTAB's s = r − αv, methods.cuh BsSIn), so
// the vector pass that would store it first is not a launch of its own; the
// epilogue stores the element for its own point.  Only transforms that read
// vectors this kernel does not write (no ping-pong needed between CTAs).
template <typename T, class Epi, class XIn = XLoad<T>, int MINB = 1, bool REALO = false, bool PREX = false>
__global__ void __launch_bounds__(256, MINB)
stencil7_kernel(const typename CT<T>::c* __restrict__ x, int nx, int ny, int nz, int z0, int nzl, int zc,
                typename CT<T>::c d, typename CT<T>::c ox, typename CT<T>::c oy, typename CT<T>::c oz,
                Epi epi, Red red, State* st, const int* gate, XIn xin) {
  using C = typename CT<T>::c;
  constexpr int KK = Epi::K > 0 ? Epi::K : 1;
  constexpr bool PLAIN = std::is_same<XIn, XLoad<T>>::value;
  if (pdl_gate(gate)) return;
  epi.load(st);
  xin.load(st);
  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);
  const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
  const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int zb = blockIdx.z * zc, ze = min(zb + zc, nzl);
  if (ix < nx && iy < ny && zb < ze) {
    // 32-bit in-plane offsets; the column pointer steps one plane per z
    const int plane = nx * ny;
    const bool hxm = ix > 0, hxp = ix < nx - 1, hym = iy > 0, hyp = iy < ny - 1;
    const C zero = czero<C>();
    // per-thread clamped offsets and coefficients of the in-plane neighbours
    const int oxm = hxm ? -1 : 0, oxq = hxp ? 1 : 0, oym = hym ? -nx : 0, oyq = hyp ? nx : 0;
    const C cxm = hxm ? ox : zero, cxq = hxp ? ox : zero, cym = hym ? oy : zero, cyq = hyp ? oy : zero;
    int zg = z0 + zb;
    const C* xp = x + (int64_t)zg * plane + ix + nx * iy;
    int64_t gi = (int64_t)zg * plane + ix + nx * iy;    // global (input) index
    int64_t li = (int64_t)zb * plane + ix + nx * iy;    // local (epilogue) index
    // lattice value at offset o from the current point
    auto X = [&](int o) -> C {
      if constexpr (PLAIN) return xp[o];
      else return xin(x, gi + o);
    };
    using EP = EpiPre<Epi>;
    // PREX: the epilogue's early load is this product's own input element
    // (chosen by the launcher from pre_src()): taken from `cur`, not loaded
    typename EP::P pnext{};
    if constexpr (!PREX) pnext = EP::pre(epi, li);   // the epilogue's inputs, a plane ahead
    C below = zg > 0 ? X(-plane) : zero;
    C cur = X(0);
#pragma unroll 2
    for (int zl = zb; zl < ze; ++zl, ++zg) {
      typename EP::P pcur = pnext;
      if constexpr (PREX) pcur = cur;
      else if (zl + 1 < ze) pnext = EP::pre(epi, li + plane);
      // every load of the plane first, then the terms in ascending column order
      C above = zero;
      if (zg < nz - 1) above = X(plane);
      const C ym = X(oym);
      const C xm = X(oxm);
      const C xq = X(oxq);
      const C yq = X(oyq);
      C acc = zero;
      st_fma<REALO>(acc, oz, below);
      st_fma<REALO>(acc, cym, ym);
      st_fma<REALO>(acc, cxm, xm);
      cfma(acc, d, cur);
      st_fma<REALO>(acc, cxq, xq);
      st_fma<REALO>(acc, cyq, yq);
      st_fma<REALO>(acc, oz, above);
      if constexpr (PLAIN && EpiWantsX<Epi>::value) epi.post_x(li, acc, pcur, cur, dacc);
      else EP::post(epi, li, acc, pcur, dacc);
      below = cur;
      cur = above;
      xp += plane;
      gi += plane;
      li += plane;
    }
  }
  if constexpr (Epi::K > 0) finish_reduction<KK, 256, Epi>(dacc, red, st);
}

// ---------------------------------------------------------------------------
// K4 fused vector pass: one grid-stride sweep applying a method-phase
// functor to every local element, with up to K fp64 partial sums.
// ---------------------------------------------------------------------------
template <int NT, class Op>
__global__ void __launch_bounds__(NT)
pass_kernel(Op op, int64_t n, Red red, State* st, const int* gate) {
  constexpr int KK = Op::K > 0 ? Op::K : 1;
  if (pdl_gate(gate)) return;
  op.load(st);
  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);
  for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) op(i, dacc);
  if constexpr (Op::K > 0) finish_reduction<KK, NT, Op>(dacc, red, st);
}

// epilogue applied as a pass over a stored vector (multi-GPU Aᴴ: after the
// reduce-scatter the epilogue runs on the local slice)
template <typename C, class Epi>
struct EpiPass {
  static constexpr int K = Epi::K;
  Epi epi;
  const C* w;
  __device__ void load(const State* st) { epi.load(st); }
  __device__ void operator()(int64_t i, double2* acc) { epi(i, w[i], acc); }
  static __device__ void finish(State* st, const double2* s) { Epi::finish(st, s); }
};

// replicated vectors: the epilogue over Σ_ranks parts[r][i] (rank order, fp64)
template <typename C, class Epi>
struct EpiPassSum {
  static constexpr int K = Epi::K;
  Epi epi;
  const C* parts;
  int world;
  int64_t n;
  __device__ void load(const State* st) { epi.load(st); }
  __device__ void operator()(int64_t i, double2* acc) {
    double2 s = make_double2(0.0, 0.0);
    for (int r = 0; r < world; ++r) {
      const C p = parts[(int64_t)r * n + i];
      s.x += (double)p.x; s.y += (double)p.y;
    }
    epi(i, fromd2<C>(s), acc);
  }
  static __device__ void finish(State* st, const double2* s) { Epi::finish(st, s); }
};

// multi-GPU scalar step: sum the world×K allgathered rank sums in rank order
template <int K, class Fin>
__global__ void scalar_kernel(const double2* all, int world, State* st, const int* gate) {
  if (pdl_gate(gate)) return;
  double2 s[K];
  for (int k = 0; k < K; ++k) s[k] = make_double2(0.0, 0.0);
  for (int r = 0; r < world; ++r)
    for (int k = 0; k < K; ++k) { s[k].x += all[r * K + k].x; s[k].y += all[r * K + k].y; }
  Fin::finish(st, s);
}

}  // namespace ccg
