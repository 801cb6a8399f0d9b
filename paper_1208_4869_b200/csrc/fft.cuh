// fft.cuh — the FFT block-Toeplitz operator: the
// matvec of a 3-level Toeplitz matrix on an nx × ny × nz lattice,
//   (A x)_i = d·x_i + Σ_{j≠i} K(r_i − r_j)·x_j,
// the structure of the discrete-dipole systems the paper was written for
// (P:47 [§1], DDSCAT; BASELINE configs 2 and 4 are scalar instances with
// K(δ) = 0.1·exp(i k|δ|)/|δ|).  The lattice sum is a linear convolution;
// embedded in a circulant of size X2 × Y2 × Z2 (each ≥ 2n − 1, a power of
// two) it becomes  y = IFFT( FFT(K_pad) ⊙ FFT(x_pad) )  restricted to the box.
//
// Five kernels per product (all line FFTs in shared memory, radix-2 stages
// fused in pairs; passes 2-4 can be one kernel, fft_yz, CCG_FFT_YZ=1):
//   fwd_x   : the ny·nz nonzero x-lines of x_pad (zero padding not read)
//   fwd_y   : the X2·nz nonzero y-lines
//   z_mul   : every (kx, ky) z-line: forward FFT, ⊙ K̂ (the mirrored entry
//             K̂(−k) for Aᵀ), inverse FFT, only z < nz stored
//   inv_y   : X2·nz y-lines, only y < ny stored
//   inv_x   : ny·nz x-lines, x < nx → + d·x, method epilogue + reduction
// Forward transforms are decimation-in-time (bit-reversed load, natural
// output), inverse ones decimation-in-frequency (natural load, bit-reversed
// output), so no explicit permutation pass is needed.  K̂ (normalised by
// 1/(X2·Y2·Z2)) is computed once on the host in double precision.
// Aᴴx = conj(Aᵀ conj x).
#pragma once
#include "common.cuh"

namespace ccg {

struct FftGeo {
  int nx, ny, nz;      // lattice
  int X2, Y2, Z2;      // padded (power-of-two) sizes
  int lx, ly, lz;      // log2 of the padded sizes
  int tyz;             // lines per CTA in the y / z passes (divides X2)
  int tx;              // lines per CTA in the x passes
};

__device__ __forceinline__ int bitrev(int v, int logL) {
  return logL == 0 ? 0 : (int)(__brev((unsigned)v) >> (32 - logL));
}

// twiddle w = exp(−2πi·m/L) (forward) or its conjugate (inverse), from the
// table tw[k] = exp(−2πi k/Lmax) of the longest axis (L divides Lmax)
template <typename C>
__device__ __forceinline__ C twiddle(const C* __restrict__ tw, int m, int stride, bool inv) {
  C w = __ldg(tw + m * stride);
  if (inv) w.y = -w.y;
  return w;
}

// In-place decimation-in-time FFT of TX lines of length L = 2^logL held in
// shared memory as buf[l·TX + t]; input in bit-reversed order, output
// natural.  Radix-2 stages are fused in pairs (each thread takes a quad of
// points through stages s and s+1 in registers: the same operations in the
// same order as two radix-2 stages, half the barriers and shared-memory
// traffic); an odd last stage runs alone.  Called by all threads of the CTA.
// Strided form: element l of line t at buf[l·ES + t·LS] (the plain form is
// ES = TX, LS = 1: lines interleaved).
template <typename C>
__device__ void fft_dit_s(C* buf, int logL, int TX, int ES, int LS, bool inv, const C* __restrict__ tw,
                          int twstride) {
  const int L = 1 << logL;
  int s = 0;
  for (; s + 1 < logL; s += 2) {
    const int h = 1 << s;
    const int nq = TX * (L >> 2);
    __syncthreads();
    for (int b = threadIdx.x; b < nq; b += blockDim.x) {
      const int t = b % TX, q = b / TX;
      const int m = q & (h - 1);
      const int i0 = ((q >> s) << (s + 2)) + m;
      const C w1 = twiddle(tw, m << (logL - s - 1), twstride, inv);
      const C w2 = twiddle(tw, m << (logL - s - 2), twstride, inv);
      const C w3 = twiddle(tw, (m + h) << (logL - s - 2), twstride, inv);
      const C x0 = buf[i0 * ES + t * LS], x1 = buf[(i0 + h) * ES + t * LS];
      const C x2 = buf[(i0 + 2 * h) * ES + t * LS], x3 = buf[(i0 + 3 * h) * ES + t * LS];
      const C p1 = cmulc(x1, w1), p3 = cmulc(x3, w1);
      const C a0 = cadd(x0, p1), a1 = csub(x0, p1), a2 = cadd(x2, p3), a3 = csub(x2, p3);
      const C q2 = cmulc(a2, w2), q3 = cmulc(a3, w3);
      buf[i0 * ES + t * LS] = cadd(a0, q2);
      buf[(i0 + 2 * h) * ES + t * LS] = csub(a0, q2);
      buf[(i0 + h) * ES + t * LS] = cadd(a1, q3);
      buf[(i0 + 3 * h) * ES + t * LS] = csub(a1, q3);
    }
  }
  if (s < logL) {                       // odd last stage
    const int h = 1 << s;
    const int nb = TX * (L >> 1);
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const int t = b % TX, q = b / TX;
      const int m = q & (h - 1);
      const int i0 = ((q >> s) << (s + 1)) + m, i1 = i0 + h;
      const C w = twiddle(tw, m << (logL - s - 1), twstride, inv);
      const C a = buf[i0 * ES + t * LS];
      const C bb = cmulc(buf[i1 * ES + t * LS], w);
      buf[i0 * ES + t * LS] = cadd(a, bb);
      buf[i1 * ES + t * LS] = csub(a, bb);
    }
  }
  __syncthreads();
}

// In-place decimation-in-frequency FFT: natural input, bit-reversed output;
// stages s = logL−1 … 0 fused in pairs (s, s−1) the same way.
template <typename C>
__device__ void fft_dif_s(C* buf, int logL, int TX, int ES, int LS, bool inv, const C* __restrict__ tw,
                          int twstride) {
  const int L = 1 << logL;
  int s = logL - 1;
  for (; s >= 1; s -= 2) {
    const int H = 1 << s, hh = H >> 1;
    const int nq = TX * (L >> 2);
    __syncthreads();
    for (int b = threadIdx.x; b < nq; b += blockDim.x) {
      const int t = b % TX, q = b / TX;
      const int m = q & (hh - 1);
      const int i0 = ((q >> (s - 1)) << (s + 1)) + m;
      const C wa = twiddle(tw, m << (logL - s - 1), twstride, inv);
      const C wb = twiddle(tw, (m + hh) << (logL - s - 1), twstride, inv);
      const C wc = twiddle(tw, m << (logL - s), twstride, inv);
      const C x0 = buf[i0 * ES + t * LS], x1 = buf[(i0 + hh) * ES + t * LS];
      const C x2 = buf[(i0 + H) * ES + t * LS], x3 = buf[(i0 + H + hh) * ES + t * LS];
      const C a0 = cadd(x0, x2), a2 = cmulc(csub(x0, x2), wa);
      const C a1 = cadd(x1, x3), a3 = cmulc(csub(x1, x3), wb);
      buf[i0 * ES + t * LS] = cadd(a0, a1);
      buf[(i0 + hh) * ES + t * LS] = cmulc(csub(a0, a1), wc);
      buf[(i0 + H) * ES + t * LS] = cadd(a2, a3);
      buf[(i0 + H + hh) * ES + t * LS] = cmulc(csub(a2, a3), wc);
    }
  }
  if (s == 0) {                         // odd last stage
    const int nb = TX * (L >> 1);
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const int t = b % TX, q = b / TX;
      const int i0 = q << 1, i1 = i0 + 1;
      const C w = twiddle(tw, 0, twstride, inv);
      const C a = buf[i0 * ES + t * LS];
      const C bb = buf[i1 * ES + t * LS];
      buf[i0 * ES + t * LS] = cadd(a, bb);
      buf[i1 * ES + t * LS] = cmulc(csub(a, bb), w);
    }
  }
  __syncthreads();
}

template <typename C>
__device__ __forceinline__ void fft_dit(C* buf, int logL, int TX, bool inv, const C* __restrict__ tw, int twstride) {
  fft_dit_s(buf, logL, TX, TX, 1, inv, tw, twstride);
}
template <typename C>
__device__ __forceinline__ void fft_dif(C* buf, int logL, int TX, bool inv, const C* __restrict__ tw, int twstride) {
  fft_dif_s(buf, logL, TX, TX, 1, inv, tw, twstride);
}

// (1) x_pad lines (y < ny, z < nz): load x (conj if CONJ_IN), zero pad, DIT along x
template <typename T, bool CONJ_IN>
__global__ void __launch_bounds__(256)
fft_fwd_x(const typename CT<T>::c* __restrict__ x, typename CT<T>::c* __restrict__ W, FftGeo g,
          const typename CT<T>::c* __restrict__ tw, int twstride, const int* gate) {
  using C = typename CT<T>::c;
  if (pdl_gate(gate)) return;
  extern __shared__ __align__(16) unsigned char fft_sm[];
  C* buf = reinterpret_cast<C*>(fft_sm);
  const int TX = g.tx, L = g.X2;
  const int nlines = g.ny * g.nz;
  const int l0 = blockIdx.x * TX;
  for (int e = threadIdx.x; e < TX * L; e += blockDim.x) {
    const int t = e / L, l = e % L;
    const int li = l0 + t;
    C v = czero<C>();
    if (li < nlines && l < g.nx) {
      v = x[(int64_t)li * g.nx + l];
      if (CONJ_IN) v.y = -v.y;
    }
    buf[bitrev(l, g.lx) * TX + t] = v;
  }
  fft_dit(buf, g.lx, TX, false, tw, twstride);
  for (int e = threadIdx.x; e < TX * L; e += blockDim.x) {
    const int t = e / L, k = e % L;
    const int li = l0 + t;
    if (li < nlines) {
      const int y = li % g.ny, z = li / g.ny;
      W[((int64_t)z * g.Y2 + y) * g.X2 + k] = buf[k * TX + t];
    }
  }
}

// (2) y lines (kx, z < nz), DIT along y (rows y ≥ ny are zero, not read)
template <typename T>
__global__ void __launch_bounds__(256)
fft_fwd_y(typename CT<T>::c* __restrict__ W, FftGeo g, const typename CT<T>::c* __restrict__ tw, int twstride,
          const int* gate) {
  using C = typename CT<T>::c;
  if (pdl_gate(gate)) return;
  extern __shared__ __align__(16) unsigned char fft_sm[];
  C* buf = reinterpret_cast<C*>(fft_sm);
  const int TX = g.tyz, L = g.Y2;
  const int kx0 = blockIdx.x * TX, z = blockIdx.y;
  C* base = W + (int64_t)z * g.Y2 * g.X2 + kx0;
  for (int e = threadIdx.x; e < TX * L; e += blockDim.x) {
    const int t = e % TX, l = e / TX;
    buf[bitrev(l, g.ly) * TX + t] = l < g.ny ? base[(int64_t)l * g.X2 + t] : czero<C>();
  }
  fft_dit(buf, g.ly, TX, false, tw, twstride);
  for (int e = threadIdx.x; e < TX * L; e += blockDim.x) {
    const int t = e % TX, k = e / TX;
    base[(int64_t)k * g.X2 + t] = buf[k * TX + t];
  }
}

// (3) z lines (kx, ky): DIT forward (z ≥ nz zero), ⊙ K̂ (mirrored for Aᵀ),
// DIF inverse, store z < nz
template <typename T, bool TRANS>
__global__ void __launch_bounds__(256)
fft_z_mul(typename CT<T>::c* __restrict__ W, const typename CT<T>::c* __restrict__ Kh, FftGeo g,
          const typename CT<T>::c* __restrict__ tw, int twstride, const int* gate) {
  using C = typename CT<T>::c;
  if (pdl_gate(gate)) return;
  extern __shared__ __align__(16) unsigned char fft_sm[];
  C* buf = reinterpret_cast<C*>(fft_sm);
  const int TX = g.tyz, L = g.Z2;
  const int kx0 = blockIdx.x * TX, ky = blockIdx.y;
  const int64_t plane = (int64_t)g.X2 * g.Y2;
  C* base = W + (int64_t)ky * g.X2 + kx0;
  for (int e = threadIdx.x; e < TX * L; e += blockDim.x) {
    const int t = e % TX, l = e / TX;
    buf[bitrev(l, g.lz) * TX + t] = l < g.nz ? base[(int64_t)l * plane + t] : czero<C>();
  }
  fft_dit(buf, g.lz, TX, false, tw, twstride);
  for (int e = threadIdx.x; e < TX * L; e += blockDim.x) {
    const int t = e % TX, k = e / TX;
    int64_t ki;
    if (TRANS) {
      const int mx = (g.X2 - (kx0 + t)) & (g.X2 - 1), my = (g.Y2 - ky) & (g.Y2 - 1), mz = (g.Z2 - k) & (g.Z2 - 1);
      ki = ((int64_t)mz * g.Y2 + my) * g.X2 + mx;
    } else {
      ki = ((int64_t)k * g.Y2 + ky) * g.X2 + kx0 + t;
    }
    buf[k * TX + t] = cmulc(buf[k * TX + t], __ldg(Kh + ki));
  }
  fft_dif(buf, g.lz, TX, true, tw, twstride);
  for (int e = threadIdx.x; e < TX * g.nz; e += blockDim.x) {
    const int t = e % TX, l = e / TX;
    base[(int64_t)l * plane + t] = buf[bitrev(l, g.lz) * TX + t];
  }
}

// (4) y lines (kx, z < nz): DIF inverse, store y < ny
template <typename T>
__global__ void __launch_bounds__(256)
fft_inv_y(typename CT<T>::c* __restrict__ W, FftGeo g, const typename CT<T>::c* __restrict__ tw, int twstride,
          const int* gate) {
  using C = typename CT<T>::c;
  if (pdl_gate(gate)) return;
  extern __shared__ __align__(16) unsigned char fft_sm[];
  C* buf = reinterpret_cast<C*>(fft_sm);
  const int TX = g.tyz, L = g.Y2;
  const int kx0 = blockIdx.x * TX, z = blockIdx.y;
  C* base = W + (int64_t)z * g.Y2 * g.X2 + kx0;
  for (int e = threadIdx.x; e < TX * L; e += blockDim.x) {
    const int t = e % TX, l = e / TX;
    buf[l * TX + t] = base[(int64_t)l * g.X2 + t];
  }
  fft_dif(buf, g.ly, TX, true, tw, twstride);
  for (int e = threadIdx.x; e < TX * g.ny; e += blockDim.x) {
    const int t = e % TX, l = e / TX;
    base[(int64_t)l * g.X2 + t] = buf[bitrev(l, g.ly) * TX + t];
  }
}

// (2-4 fused, opt-in: measured neutral) one kx plane per CTA, whole in shared
// memory as P[y][z] (row stride RS = Z2 + 1: the z-line pass reads rows 16 B
// apart, conflict-free): y DIT over the nz nonzero z-lines (bit-reversed load),
// z DIF forward (natural in, bit-reversed kz out) ⊙ K̂ (mirrored for Aᵀ), z
// DIT inverse (bit-reversed in, natural out), y DIF inverse over z < nz; stores
// y < ny, z < nz.  The same transforms as passes (2)-(4) with no round trip
// of the work array through L2 and two launches fewer per product.
template <typename T, bool TRANS>
__global__ void __launch_bounds__(512)
fft_yz(typename CT<T>::c* __restrict__ W, const typename CT<T>::c* __restrict__ Kh, FftGeo g,
       const typename CT<T>::c* __restrict__ tw, int twy, int twz, const int* gate) {
  using C = typename CT<T>::c;
  if (pdl_gate(gate)) return;
  extern __shared__ __align__(16) unsigned char fft_sm[];
  C* P = reinterpret_cast<C*>(fft_sm);
  const int kx = blockIdx.x;
  const int RS = g.Z2 + 1;
  const int64_t sz = (int64_t)g.Y2 * g.X2;
  for (int e = threadIdx.x; e < g.Y2 * g.Z2; e += blockDim.x) {
    const int z = e / g.Y2, y = e % g.Y2;
    C v = czero<C>();
    if (y < g.ny && z < g.nz) v = W[(int64_t)z * sz + (int64_t)y * g.X2 + kx];
    P[bitrev(y, g.ly) * RS + z] = v;
  }
  fft_dit_s(P, g.ly, g.nz, RS, 1, false, tw, twy);
  fft_dif_s(P, g.lz, g.Y2, 1, RS, false, tw, twz);
  for (int e = threadIdx.x; e < g.Y2 * g.Z2; e += blockDim.x) {
    const int ky = e / g.Z2, p = e % g.Z2;
    const int kz = bitrev(p, g.lz);
    int64_t ki;
    if (TRANS) {
      const int mx = (g.X2 - kx) & (g.X2 - 1), my = (g.Y2 - ky) & (g.Y2 - 1), mz = (g.Z2 - kz) & (g.Z2 - 1);
      ki = ((int64_t)mz * g.Y2 + my) * g.X2 + mx;
    } else {
      ki = ((int64_t)kz * g.Y2 + ky) * g.X2 + kx;
    }
    P[ky * RS + p] = cmulc(P[ky * RS + p], __ldg(Kh + ki));
  }
  fft_dit_s(P, g.lz, g.Y2, 1, RS, true, tw, twz);
  fft_dif_s(P, g.ly, g.nz, RS, 1, true, tw, twy);
  for (int e = threadIdx.x; e < g.ny * g.nz; e += blockDim.x) {
    const int z = e / g.ny, y = e % g.ny;
    W[(int64_t)z * sz + (int64_t)y * g.X2 + kx] = P[bitrev(y, g.ly) * RS + z];
  }
}

// (5) x lines (y < ny, z < nz): DIF inverse; x < nx: v (conj if CONJ) + d·x_i
// → method epilogue on the rows this rank owns, [row0, row0 + nloc)
template <typename T, bool CONJ, class Epi>
__global__ void __launch_bounds__(256)
fft_inv_x(const typename CT<T>::c* __restrict__ W, const typename CT<T>::c* __restrict__ x, FftGeo g,
          const typename CT<T>::c* __restrict__ tw, int twstride, typename CT<T>::c d, int64_t row0, int64_t nloc,
          Epi epi, Red red, State* st, const int* gate) {
  using C = typename CT<T>::c;
  constexpr int KK = Epi::K > 0 ? Epi::K : 1;
  if (pdl_gate(gate)) return;
  epi.load(st);
  extern __shared__ __align__(16) unsigned char fft_sm[];
  C* buf = reinterpret_cast<C*>(fft_sm);
  double2 dacc[KK];
#pragma unroll
  for (int k = 0; k < KK; ++k) dacc[k] = make_double2(0.0, 0.0);
  const int TX = g.tx, L = g.X2;
  const int nlines = g.ny * g.nz;
  const int l0 = blockIdx.x * TX;
  for (int e = threadIdx.x; e < TX * L; e += blockDim.x) {
    const int t = e / L, l = e % L;
    const int li = l0 + t;
    if (li < nlines) {
      const int y = li % g.ny, z = li / g.ny;
      buf[l * TX + t] = W[((int64_t)z * g.Y2 + y) * g.X2 + l];
    }
  }
  fft_dif(buf, g.lx, TX, true, tw, twstride);
  for (int e = threadIdx.x; e < TX * g.nx; e += blockDim.x) {
    const int t = e / g.nx, l = e % g.nx;
    const int li = l0 + t;
    if (li < nlines) {
      const int64_t gi = (int64_t)li * g.nx + l;
      if (gi >= row0 && gi < row0 + nloc) {
        C v = buf[bitrev(l, g.lx) * TX + t];
        if (CONJ) v.y = -v.y;
        const C xi = x[gi];
        C dx = czero<C>();
        cfma(dx, d, xi);
        epi(gi - row0, cadd(v, dx), dacc);
      }
    }
  }
  if constexpr (Epi::K > 0) finish_reduction<KK, 256, Epi>(dacc, red, st);
}

}  // namespace ccg
