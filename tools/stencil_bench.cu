// stencil_bench.cu — standalone microbenchmark of 7-point stencil kernel
// layouts for config 5 (128³ c128, BJ:11).  Development tool, not part of
// libccg.so: each variant computes y = A·x with the library's term order
// (oz·below, oy·(y−1), ox·(x−1), d·cur, ox·(x+1), oy·(y+1), oz·above), so
// every variant must be bitwise equal to the simple one.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -I paper_1208_4869_b200/csrc tools/stencil_bench.cu -o /tmp/stencil_bench
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "bulk.cuh"

using namespace ccg;
using C = double2;

__device__ __forceinline__ void term(C& acc, C coef, C v) {
  C p = czero<C>();
  cfma(p, coef, v);
  acc = cadd(acc, p);
}

struct Co { C d, ox, oy, oz; };

// V0: the library kernel (z-march, zc planes per thread, neighbours via __ldg)
__global__ void __launch_bounds__(256) v0_march(const C* __restrict__ x, C* __restrict__ y, int nx, int ny, int nz,
                                                int zc, Co k) {
  const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
  const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int zb = blockIdx.z * zc, ze = min(zb + zc, nz);
  const int64_t plane = (int64_t)nx * ny;
  if (ix >= nx || iy >= ny) return;
  const int64_t col = ix + (int64_t)nx * iy;
  C below = zb > 0 ? __ldg(x + col + plane * (zb - 1)) : czero<C>();
  C cur = __ldg(x + col + plane * zb);
  for (int z = zb; z < ze; ++z) {
    const int64_t gi = col + plane * z;
    const C above = z < nz - 1 ? __ldg(x + gi + plane) : czero<C>();
    C acc = czero<C>();
    if (z > 0) term(acc, k.oz, below);
    if (iy > 0) term(acc, k.oy, __ldg(x + gi - nx));
    if (ix > 0) term(acc, k.ox, __ldg(x + gi - 1));
    term(acc, k.d, cur);
    if (ix < nx - 1) term(acc, k.ox, __ldg(x + gi + 1));
    if (iy < ny - 1) term(acc, k.oy, __ldg(x + gi + nx));
    if (z < nz - 1) term(acc, k.oz, above);
    y[gi] = acc;
    below = cur;
    cur = above;
  }
}

// V3: one thread per point, 7 loads
__global__ void __launch_bounds__(256) v3_point(const C* __restrict__ x, C* __restrict__ y, int nx, int ny, int nz,
                                                Co k) {
  const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
  const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int z = blockIdx.z;
  if (ix >= nx || iy >= ny) return;
  const int64_t plane = (int64_t)nx * ny;
  const int64_t gi = ix + (int64_t)nx * iy + plane * z;
  const C b = z > 0 ? __ldg(x + gi - plane) : czero<C>();
  const C ym = iy > 0 ? __ldg(x + gi - nx) : czero<C>();
  const C xm = ix > 0 ? __ldg(x + gi - 1) : czero<C>();
  const C c = __ldg(x + gi);
  const C xp = ix < nx - 1 ? __ldg(x + gi + 1) : czero<C>();
  const C yp = iy < ny - 1 ? __ldg(x + gi + nx) : czero<C>();
  const C a = z < nz - 1 ? __ldg(x + gi + plane) : czero<C>();
  C acc = czero<C>();
  if (z > 0) term(acc, k.oz, b);
  if (iy > 0) term(acc, k.oy, ym);
  if (ix > 0) term(acc, k.ox, xm);
  term(acc, k.d, c);
  if (ix < nx - 1) term(acc, k.ox, xp);
  if (iy < ny - 1) term(acc, k.oy, yp);
  if (z < nz - 1) term(acc, k.oz, a);
  y[gi] = acc;
}

__device__ __forceinline__ C shfl(C v, int src) {
  C r;
  r.x = __shfl_sync(0xffffffffu, v.x, src);
  r.y = __shfl_sync(0xffffffffu, v.y, src);
  return r;
}

// V1: z-march, ZC planes, x±1 through warp shuffles (edge lanes load), the
// plane two ahead prefetched (register queue below/cur/above/next2), the y±1
// rows of the current plane loaded at the top of the step.
template <int ZC>
__global__ void __launch_bounds__(256) v1_march_shfl(const C* __restrict__ x, C* __restrict__ y, int nx, int ny,
                                                     int nz, Co k) {
  const int lane = threadIdx.x & 31;
  const int ix = blockIdx.x * 32 + lane;
  const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int zb = blockIdx.z * ZC, ze = min(zb + ZC, nz);
  const int64_t plane = (int64_t)nx * ny;
  const bool in = ix < nx && iy < ny;
  const int64_t col = min(ix, nx - 1) + (int64_t)nx * min(iy, ny - 1);
  C below = (in && zb > 0) ? __ldg(x + col + plane * (zb - 1)) : czero<C>();
  C cur = in ? __ldg(x + col + plane * zb) : czero<C>();
  C above = (in && zb + 1 < nz) ? __ldg(x + col + plane * (zb + 1)) : czero<C>();
#pragma unroll 4
  for (int z = zb; z < ze; ++z) {
    const int64_t gi = col + plane * z;
    const C next2 = (in && z + 2 < nz && z + 2 <= ze) ? __ldg(x + gi + 2 * plane) : czero<C>();
    const C ym = (in && iy > 0) ? __ldg(x + gi - nx) : czero<C>();
    const C yp = (in && iy < ny - 1) ? __ldg(x + gi + nx) : czero<C>();
    C xm = shfl(cur, (lane + 31) & 31), xp = shfl(cur, (lane + 1) & 31);
    if (lane == 0) xm = (in && ix > 0) ? __ldg(x + gi - 1) : czero<C>();
    if (lane == 31) xp = (in && ix < nx - 1) ? __ldg(x + gi + 1) : czero<C>();
    if (in) {
      C acc = czero<C>();
      if (z > 0) term(acc, k.oz, below);
      if (iy > 0) term(acc, k.oy, ym);
      if (ix > 0) term(acc, k.ox, xm);
      term(acc, k.d, cur);
      if (ix < nx - 1) term(acc, k.ox, xp);
      if (iy < ny - 1) term(acc, k.oy, yp);
      if (z < nz - 1) term(acc, k.oz, above);
      y[gi] = acc;
    }
    below = cur;
    cur = above;
    above = next2;
  }
}

// V2: 2.5-D shared-memory tiling.  CTA = 32 (x) × 8 (y) outputs marching ZC
// planes; a ring of S halo'd plane tiles (34 × 10) filled with cp.async (16 B
// per element); one barrier per plane.
template <int ZC, int S>
__global__ void __launch_bounds__(256) v2_smem(const C* __restrict__ x, C* __restrict__ y, int nx, int ny, int nz,
                                               Co k) {
  constexpr int TX = 34, TY = 10, TE = TX * TY;   // 340 elements per stage
  __shared__ __align__(16) C tile[S][TE];
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * 32 - 1, y0 = blockIdx.y * 8 - 1;
  const int zb = blockIdx.z * ZC, ze = min(zb + ZC, nz);
  const int64_t plane = (int64_t)nx * ny;
  // load plane zz into slot
  auto load = [&](int zz, int slot) {
    for (int e = t; e < TE; e += 256) {
      const int tx = e % TX, ty = e / TX;
      const int gx = x0 + tx, gy = y0 + ty;
      C* dst = &tile[slot][e];
      if (zz >= 0 && zz < nz && gx >= 0 && gx < nx && gy >= 0 && gy < ny) {
        const C* src = x + gx + (int64_t)nx * gy + plane * zz;
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src));
      } else {
        *dst = czero<C>();
      }
    }
  };
  // prologue: planes zb-1 .. zb+S-3 (S-1 planes)
  for (int s = 0; s < S - 1; ++s) {
    load(zb - 1 + s, s);
    asm volatile("cp.async.commit_group;");
  }
  const int lx = (t & 31) + 1, ly = (t >> 5) + 1;
  const int ix = x0 + lx, iy = y0 + ly;
  for (int z = zb; z < ze; ++z) {
    // issue plane z + S - 2 (slot of plane z - 2, free after the last barrier)
    const int zi = z + S - 2;
    load(zi, (zi - zb + 1) % S);
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 3));   // planes ≤ z+1 landed (this thread's)
    __syncthreads();
    const C* pb = tile[(z - zb) % S];        // plane z-1
    const C* pc = tile[(z - zb + 1) % S];    // plane z
    const C* pa = tile[(z - zb + 2) % S];    // plane z+1
    if (ix < nx && iy < ny) {
      const int e = lx + TX * ly;
      C acc = czero<C>();
      if (z > 0) term(acc, k.oz, pb[e]);
      if (iy > 0) term(acc, k.oy, pc[e - TX]);
      if (ix > 0) term(acc, k.ox, pc[e - 1]);
      term(acc, k.d, pc[e]);
      if (ix < nx - 1) term(acc, k.ox, pc[e + 1]);
      if (iy < ny - 1) term(acc, k.oy, pc[e + TX]);
      if (z < nz - 1) term(acc, k.oz, pa[e]);
      y[ix + (int64_t)nx * iy + plane * z] = acc;
    }
    __syncthreads();
  }
  asm volatile("cp.async.wait_all;");
}

// V4: z-march, each thread 2 rows (iy, iy+1): the rows share their y
// neighbour loads; x±1 by shuffles; block 32 × 4 threads = 32 × 8 points.
template <int ZC>
__global__ void __launch_bounds__(128) v4_march2(const C* __restrict__ x, C* __restrict__ y, int nx, int ny, int nz,
                                                 Co k) {
  const int lane = threadIdx.x & 31;
  const int ix = blockIdx.x * 32 + lane;
  const int iy0 = blockIdx.y * 8 + 2 * (threadIdx.x >> 5);
  const int zb = blockIdx.z * ZC, ze = min(zb + ZC, nz);
  const int64_t plane = (int64_t)nx * ny;
  const bool inx = ix < nx;
  const int cx = min(ix, nx - 1);
  C b[2], c[2], a[2];
  for (int r = 0; r < 2; ++r) {
    const int iy = min(iy0 + r, ny - 1);
    const int64_t col = cx + (int64_t)nx * iy;
    b[r] = zb > 0 ? __ldg(x + col + plane * (zb - 1)) : czero<C>();
    c[r] = __ldg(x + col + plane * zb);
  }
  for (int z = zb; z < ze; ++z) {
    const int64_t base = cx + plane * z;
    for (int r = 0; r < 2; ++r) {
      const int iy = min(iy0 + r, ny - 1);
      a[r] = z < nz - 1 ? __ldg(x + base + (int64_t)nx * iy + plane) : czero<C>();
    }
    const C ym = iy0 > 0 ? __ldg(x + base + (int64_t)nx * (iy0 - 1)) : czero<C>();
    const C yp = iy0 + 2 < ny ? __ldg(x + base + (int64_t)nx * (iy0 + 2)) : czero<C>();
    for (int r = 0; r < 2; ++r) {
      const int iy = iy0 + r;
      C xm = shfl(c[r], (lane + 31) & 31), xp = shfl(c[r], (lane + 1) & 31);
      if (lane == 0) xm = ix > 0 ? __ldg(x + base + (int64_t)nx * min(iy, ny - 1) - 1) : czero<C>();
      if (lane == 31) xp = ix < nx - 1 ? __ldg(x + base + (int64_t)nx * min(iy, ny - 1) + 1) : czero<C>();
      if (inx && iy < ny) {
        const C yy0 = r == 0 ? ym : c[0];
        const C yy1 = r == 0 ? c[1] : yp;
        C acc = czero<C>();
        if (z > 0) term(acc, k.oz, b[r]);
        if (iy > 0) term(acc, k.oy, yy0);
        if (ix > 0) term(acc, k.ox, xm);
        term(acc, k.d, c[r]);
        if (ix < nx - 1) term(acc, k.ox, xp);
        if (iy < ny - 1) term(acc, k.oy, yy1);
        if (z < nz - 1) term(acc, k.oz, a[r]);
        y[base + (int64_t)nx * iy] = acc;
      }
    }
    for (int r = 0; r < 2; ++r) { b[r] = c[r]; c[r] = a[r]; }
  }
}

// V5: TMA bulk copies of contiguous plane slabs.  CTA = TY full rows (x is
// the whole row, so a slab of TY+2 rows of one plane is ONE contiguous range)
// marching ZC planes through a ring of S slab stages (mbarrier tx-count per
// stage); 256 threads compute TY·nx outputs per plane from shared memory, the
// z neighbours from the adjacent stages; one barrier per plane frees the
// stage of plane z−1 for the bulk copy of plane z+S−1.
template <int TY, int ZC, int S>
__global__ void __launch_bounds__(256) v5_bulk(const C* __restrict__ x, C* __restrict__ y, int nx, int ny, int nz,
                                               Co k) {
  extern __shared__ __align__(128) unsigned char sm_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm_raw);
  C* stage = reinterpret_cast<C*>(sm_raw + 128);
  const int SE = (TY + 2) * nx;              // elements per stage (row -1 .. TY)
  const int t = threadIdx.x;
  const int y0 = blockIdx.x * TY;
  const int zb = blockIdx.y * ZC, ze = min(zb + ZC, nz);
  const int64_t plane = (int64_t)nx * ny;
  const int ylo = max(y0 - 1, 0), yhi = min(y0 + TY + 1, ny);     // rows present in a slab
  const uint32_t bytes = (uint32_t)((yhi - ylo) * nx * sizeof(C));
  if (t == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  // plane p (zb-1 <= p <= ze) lives in slot (p - zb + 1) % S, use (p - zb + 1) / S
  auto issue = [&](int p) {
    if (p > ze) return;                   // never waited on
    const int q = p - zb + 1;
    uint64_t* b = &bar[q % S];
    if (p < 0 || p >= nz) {               // outside the lattice: complete the phase, no data
      mbar_arrive(b);
      return;
    }
    mbar_arrive_expect_tx(b, bytes);
    bulk_g2s(stage + (size_t)(q % S) * SE + (ylo - (y0 - 1)) * nx, x + plane * p + (int64_t)ylo * nx, bytes, b, pol);
  };
  auto wait = [&](int p) {
    if (p < 0 || p >= nz) return;
    const int q = p - zb + 1;
    mbar_wait(&bar[q % S], (q / S) & 1);
  };
  if (t == 0)
    for (int p = zb - 1; p < zb - 1 + S; ++p) issue(p);
  wait(zb - 1);
  wait(zb);
  const int per = (TY * nx) / 256;   // outputs per thread per plane (nx·TY multiple of 256)
  for (int z = zb; z < ze; ++z) {
    wait(z + 1);
    const C* pb = stage + (size_t)((z - zb) % S) * SE + nx;        // row 0 of plane z-1
    const C* pc = stage + (size_t)((z - zb + 1) % S) * SE + nx;    // plane z
    const C* pa = stage + (size_t)((z - zb + 2) % S) * SE + nx;    // plane z+1
    for (int j = 0; j < per; ++j) {
      const int i = t + 256 * j;
      const int ix = i % nx, ly = i / nx, iy = y0 + ly;
      if (iy >= ny) continue;
      C acc = czero<C>();
      if (z > 0) term(acc, k.oz, pb[i]);
      if (iy > 0) term(acc, k.oy, pc[i - nx]);
      if (ix > 0) term(acc, k.ox, pc[i - 1]);
      term(acc, k.d, pc[i]);
      if (ix < nx - 1) term(acc, k.ox, pc[i + 1]);
      if (iy < ny - 1) term(acc, k.oy, pc[i + nx]);
      if (z < nz - 1) term(acc, k.oz, pa[i]);
      y[plane * z + (int64_t)y0 * nx + i] = acc;
    }
    __syncthreads();                      // every thread is done with plane z-1's stage
    if (t == 0) issue(z + S - 1);         // into the slot of plane z-1
  }
}

// FMA-accumulated term (acc += coef·v with 4 FMAs, no separate product)
__device__ __forceinline__ void mac(C& acc, C coef, C v) { cfma(acc, coef, v); }

// V3f: reference for the FMA-accumulated order
__global__ void __launch_bounds__(256) v3f_point(const C* __restrict__ x, C* __restrict__ y, int nx, int ny, int nz,
                                                 Co k) {
  const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
  const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int z = blockIdx.z;
  if (ix >= nx || iy >= ny) return;
  const int64_t plane = (int64_t)nx * ny;
  const int64_t gi = ix + (int64_t)nx * iy + plane * z;
  C acc = czero<C>();
  if (z > 0) mac(acc, k.oz, x[gi - plane]);
  if (iy > 0) mac(acc, k.oy, x[gi - nx]);
  if (ix > 0) mac(acc, k.ox, x[gi - 1]);
  mac(acc, k.d, x[gi]);
  if (ix < nx - 1) mac(acc, k.ox, x[gi + 1]);
  if (iy < ny - 1) mac(acc, k.oy, x[gi + nx]);
  if (z < nz - 1) mac(acc, k.oz, x[gi + plane]);
  y[gi] = acc;
}

// V6: z-march with ZC compile-time planes, FMA accumulation, masked loads
// (outside the lattice -> 0, terms unconditional), 32-bit in-slab offsets.
template <int ZC>
__global__ void __launch_bounds__(256) v6_march(const C* __restrict__ x, C* __restrict__ y, int nx, int ny, int nz,
                                                Co k) {
  const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
  const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int zb = blockIdx.z * ZC;
  if (ix >= nx || iy >= ny) return;
  const int plane = nx * ny;
  const C zero = czero<C>();
  const bool hxm = ix > 0, hxp = ix < nx - 1, hym = iy > 0, hyp = iy < ny - 1;
  const C* xp = x + (int64_t)zb * plane + ix + nx * iy;   // this column at plane zb
  C* yp = y + (int64_t)zb * plane + ix + nx * iy;
  C below = zb > 0 ? xp[-plane] : zero;
  C cur = xp[0];
#pragma unroll
  for (int j = 0; j < ZC; ++j) {
    const int z = zb + j;
    if (z >= nz) break;
    const C above = z < nz - 1 ? xp[plane] : zero;
    const C ym = hym ? xp[-nx] : zero;
    const C xm = hxm ? xp[-1] : zero;
    const C xq = hxp ? xp[1] : zero;
    const C yq = hyp ? xp[nx] : zero;
    C acc = zero;
    mac(acc, k.oz, below);
    mac(acc, k.oy, ym);
    mac(acc, k.ox, xm);
    mac(acc, k.d, cur);
    mac(acc, k.ox, xq);
    mac(acc, k.oy, yq);
    mac(acc, k.oz, above);
    yp[0] = acc;
    below = cur;
    cur = above;
    xp += plane;
    yp += plane;
  }
}

// V7: V6 with R rows per thread (the rows share the y-neighbour loads:
// R + 2 row loads per plane for R outputs instead of 3R); block 32 × (8/R).
template <int ZC, int R>
__global__ void __launch_bounds__(256 / R) v7_march_rows(const C* __restrict__ x, C* __restrict__ y, int nx, int ny,
                                                        int nz, Co k) {
  const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
  const int iy0 = blockIdx.y * 8 + R * (threadIdx.x >> 5);
  const int zb = blockIdx.z * ZC;
  if (ix >= nx || iy0 >= ny) return;
  const int plane = nx * ny;
  const C zero = czero<C>();
  const bool hxm = ix > 0, hxp = ix < nx - 1;
  const C* xp = x + (int64_t)zb * plane + ix + nx * iy0;
  C* yp = y + (int64_t)zb * plane + ix + nx * iy0;
  C below[R], cur[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool in = iy0 + r < ny;
    below[r] = (in && zb > 0) ? xp[r * nx - plane] : zero;
    cur[r] = in ? xp[r * nx] : zero;
  }
#pragma unroll
  for (int j = 0; j < ZC; ++j) {
    const int z = zb + j;
    if (z >= nz) break;
    C above[R];
#pragma unroll
    for (int r = 0; r < R; ++r) above[r] = (z < nz - 1 && iy0 + r < ny) ? xp[r * nx + plane] : zero;
    const C ym = iy0 > 0 ? xp[-nx] : zero;
    const C yq = iy0 + R < ny ? xp[R * nx] : zero;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (iy0 + r >= ny) break;
      const C xm = hxm ? xp[r * nx - 1] : zero;
      const C xq = hxp ? xp[r * nx + 1] : zero;
      C acc = zero;
      mac(acc, k.oz, below[r]);
      mac(acc, k.oy, r == 0 ? ym : cur[r - 1]);
      mac(acc, k.ox, xm);
      mac(acc, k.d, cur[r]);
      mac(acc, k.ox, xq);
      mac(acc, k.oy, r == R - 1 ? yq : cur[r + 1]);
      mac(acc, k.oz, above[r]);
      yp[r * nx] = acc;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) { below[r] = cur[r]; cur[r] = above[r]; }
    xp += plane;
    yp += plane;
  }
}

// V9: V6 with a register queue of the next PD "above" planes (loads issued
// PD planes ahead: PD + 4 loads in flight per thread instead of ~1 from HBM),
// MINB CTAs/SM requested in the launch bounds.
template <int ZC, int PD, int MINB>
__global__ void __launch_bounds__(256, MINB) v9_prefetch(const C* __restrict__ x, C* __restrict__ y, int nx, int ny,
                                                       int nz, Co k) {
  const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
  const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int zb = blockIdx.z * ZC;
  if (ix >= nx || iy >= ny) return;
  const int plane = nx * ny;
  const C zero = czero<C>();
  const bool hxm = ix > 0, hxp = ix < nx - 1, hym = iy > 0, hyp = iy < ny - 1;
  const C* xp = x + (int64_t)zb * plane + ix + nx * iy;
  C* yp = y + (int64_t)zb * plane + ix + nx * iy;
  C below = zb > 0 ? xp[-plane] : zero;
  C cur = xp[0];
  C q[PD];   // q[d] = plane zb + 1 + d (zero outside the lattice)
#pragma unroll
  for (int d = 0; d < PD; ++d) q[d] = zb + 1 + d < nz ? xp[(d + 1) * plane] : zero;
#pragma unroll
  for (int j = 0; j < ZC; ++j) {
    const int z = zb + j;
    if (z >= nz) break;
    const C above = q[0];
#pragma unroll
    for (int d = 0; d + 1 < PD; ++d) q[d] = q[d + 1];
    q[PD - 1] = (j + 1 + PD < ZC + 1 && z + 1 + PD < nz) ? xp[(1 + PD) * plane] : zero;
    const C ym = hym ? xp[-nx] : zero;
    const C xm = hxm ? xp[-1] : zero;
    const C xq = hxp ? xp[1] : zero;
    const C yq = hyp ? xp[nx] : zero;
    C acc = zero;
    mac(acc, k.oz, below);
    mac(acc, k.oy, ym);
    mac(acc, k.ox, xm);
    mac(acc, k.d, cur);
    mac(acc, k.ox, xq);
    mac(acc, k.oy, yq);
    mac(acc, k.oz, above);
    yp[0] = acc;
    below = cur;
    cur = above;
    xp += plane;
    yp += plane;
  }
}

// ---- with a BiCGSTAB BsT-like epilogue: t = A s stored, fp64 partials
// <t,s> and ||t||^2, per-CTA slot + arrival ticket, the last CTA sums the
// slots in order (the library's finish_reduction pattern)
struct EpiOut { double2* part; unsigned* ticket; double2* result; };

template <bool REL = false>
__device__ __forceinline__ void epi_finish(double2 a0, double2 a1, EpiOut e, unsigned bid, unsigned nb) {
  __shared__ double2 sm[8][2];
  __shared__ int last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    a0.x += __shfl_xor_sync(~0u, a0.x, o); a0.y += __shfl_xor_sync(~0u, a0.y, o);
    a1.x += __shfl_xor_sync(~0u, a1.x, o); a1.y += __shfl_xor_sync(~0u, a1.y, o);
  }
  if (lane == 0) { sm[warp][0] = a0; sm[warp][1] = a1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 s0 = make_double2(0, 0), s1 = make_double2(0, 0);
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) { s0.x += sm[w][0].x; s0.y += sm[w][0].y; s1.x += sm[w][1].x; }
    e.part[2 * bid] = s0; e.part[2 * bid + 1] = s1;
    if (REL) {   // release RMW: orders this CTA's partials before its arrival, no L1 flush
      unsigned t;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(e.ticket) : "memory");
      last = t == nb - 1;
    } else {
      __threadfence();
      last = atomicAdd(e.ticket, 1u) == nb - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  if (REL) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  else __threadfence();
  double2 s0 = make_double2(0, 0), s1 = make_double2(0, 0);
  for (unsigned b = threadIdx.x; b < nb; b += blockDim.x) {
    const double2 p0 = __ldcg(e.part + 2 * b), p1 = __ldcg(e.part + 2 * b + 1);
    s0.x += p0.x; s0.y += p0.y; s1.x += p1.x;
  }
  for (int o = 16; o; o >>= 1) {
    s0.x += __shfl_xor_sync(~0u, s0.x, o); s0.y += __shfl_xor_sync(~0u, s0.y, o); s1.x += __shfl_xor_sync(~0u, s1.x, o);
  }
  __syncthreads();
  if (lane == 0) { sm[warp][0] = s0; sm[warp][1] = s1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 r0 = make_double2(0, 0), r1 = make_double2(0, 0);
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) { r0.x += sm[w][0].x; r0.y += sm[w][0].y; r1.x += sm[w][1].x; }
    e.result[0] = r0; e.result[1] = r1;
    *e.ticket = 0;
  }
}

__device__ __forceinline__ void epi_acc(double2& a0, double2& a1, C t, C s) {
  a0.x = fma(t.x, s.x, fma(t.y, s.y, a0.x));   // conj(t)·s
  a0.y = fma(t.x, s.y, fma(-t.y, s.x, a0.y));
  a1.x = fma(t.x, t.x, fma(t.y, t.y, a1.x));
}

// one z-marching tile (32 x 8 columns, ZC planes), BsT-like epilogue
template <int ZC>
__device__ __forceinline__ void tile_e(const C* __restrict__ x, C* __restrict__ y, int nx, int ny, int nz, Co k,
                                       int bx, int by, int bz, double2& a0, double2& a1) {
  const int ix = bx * 32 + (threadIdx.x & 31);
  const int iy = by * 8 + (threadIdx.x >> 5);
  const int zb = bz * ZC;
  if (ix >= nx || iy >= ny) return;
  const int plane = nx * ny;
  const C zero = czero<C>();
  const bool hxm = ix > 0, hxp = ix < nx - 1, hym = iy > 0, hyp = iy < ny - 1;
  const C* xp = x + (int64_t)zb * plane + ix + nx * iy;
  C* yp = y + (int64_t)zb * plane + ix + nx * iy;
  C below = zb > 0 ? xp[-plane] : zero;
  C cur = xp[0];
#pragma unroll
  for (int j = 0; j < ZC; ++j) {
    const int z = zb + j;
    if (z >= nz) break;
    const C above = z < nz - 1 ? xp[plane] : zero;
    const C ym = hym ? xp[-nx] : zero;
    const C xm = hxm ? xp[-1] : zero;
    const C xq = hxp ? xp[1] : zero;
    const C yq = hyp ? xp[nx] : zero;
    C acc = zero;
    mac(acc, k.oz, below);
    mac(acc, k.oy, ym);
    mac(acc, k.ox, xm);
    mac(acc, k.d, cur);
    mac(acc, k.ox, xq);
    mac(acc, k.oy, yq);
    mac(acc, k.oz, above);
    yp[0] = acc;
    epi_acc(a0, a1, acc, cur);
    below = cur;
    cur = above;
    xp += plane;
    yp += plane;
  }
}

// V10: one tile per CTA + epilogue (the library's structure)
template <int ZC, bool REL = false>
__global__ void __launch_bounds__(256) v10_epi(const C* __restrict__ x, C* __restrict__ y, int nx, int ny, int nz, Co k,
                                               EpiOut e) {
  double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
  tile_e<ZC>(x, y, nx, ny, nz, k, blockIdx.x, blockIdx.y, blockIdx.z, a0, a1);
  epi_finish<REL>(a0, a1, e, blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z),
             gridDim.x * gridDim.y * gridDim.z);
}

// V11: persistent — grid = SMs x occupancy, each CTA walks tiles (z fastest
// within a column block so consecutive tiles of a CTA share L2 lines)
template <int ZC, int MINB, bool REL = false>
__global__ void __launch_bounds__(256, MINB) v11_persist(const C* __restrict__ x, C* __restrict__ y, int nx, int ny,
                                                       int nz, Co k, EpiOut e) {
  double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
  const int tx = (nx + 31) / 32, ty = (ny + 7) / 8, tz = (nz + ZC - 1) / ZC;
  const int ntiles = tx * ty * tz;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int bx = t % tx, by = (t / tx) % ty, bz = t / (tx * ty);
    tile_e<ZC>(x, y, nx, ny, nz, k, bx, by, bz, a0, a1);
  }
  epi_finish<REL>(a0, a1, e, blockIdx.x, gridDim.x);
}

// V12: v10 without the arrival ticket (block sum + slot store only); V13: the
// epilogue arithmetic only (no block sum) — to split the epilogue's cost
template <int ZC, int MODE>
__global__ void __launch_bounds__(256) v12_parts(const C* __restrict__ x, C* __restrict__ y, int nx, int ny, int nz,
                                                 Co k, EpiOut e) {
  double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
  tile_e<ZC>(x, y, nx, ny, nz, k, blockIdx.x, blockIdx.y, blockIdx.z, a0, a1);
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (MODE == 1) {   // arithmetic only
    if (a0.x == 12345.678) e.part[bid] = a1;
    return;
  }
  __shared__ double2 sm[8][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    a0.x += __shfl_xor_sync(~0u, a0.x, o); a0.y += __shfl_xor_sync(~0u, a0.y, o);
    a1.x += __shfl_xor_sync(~0u, a1.x, o);
  }
  if (lane == 0) { sm[warp][0] = a0; sm[warp][1] = a1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 s0 = make_double2(0, 0), s1 = make_double2(0, 0);
    for (int w = 0; w < 8; ++w) { s0.x += sm[w][0].x; s0.y += sm[w][0].y; s1.x += sm[w][1].x; }
    e.part[2 * bid] = s0; e.part[2 * bid + 1] = s1;
  }
}

// V14: v10 with a two-level arrival: groups of 32 CTAs each have their own
// ticket (different L2 slices, so the same-address atomics do not serialise
// over the whole grid); the last CTA of a group sums its 32 slots with one
// warp into a group slot, and only those take the grid ticket; the last one
// sums the group slots.  Fixed order at both levels (deterministic).
struct EpiOut2 { double2* part; double2* gpart; unsigned* gticket; unsigned* ticket; double2* result; };

__device__ __forceinline__ double2 warp_sum2(double2 v) {
  for (int o = 16; o; o >>= 1) { v.x += __shfl_xor_sync(~0u, v.x, o); v.y += __shfl_xor_sync(~0u, v.y, o); }
  return v;
}

template <int ZC>
__global__ void __launch_bounds__(256) v14_epi2(const C* __restrict__ x, C* __restrict__ y, int nx, int ny, int nz,
                                                Co k, EpiOut2 e) {
  double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
  tile_e<ZC>(x, y, nx, ny, nz, k, blockIdx.x, blockIdx.y, blockIdx.z, a0, a1);
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
  __shared__ double2 sm[8][2];
  __shared__ int flag;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a0 = warp_sum2(a0);
  a1 = warp_sum2(a1);
  if (lane == 0) { sm[warp][0] = a0; sm[warp][1] = a1; }
  __syncthreads();
  const unsigned g = bid / 32, ng = (nb + 31) / 32, gs = min(32u, nb - g * 32);
  if (threadIdx.x == 0) {
    double2 s0 = make_double2(0, 0), s1 = make_double2(0, 0);
    for (int w = 0; w < 8; ++w) { s0.x += sm[w][0].x; s0.y += sm[w][0].y; s1.x += sm[w][1].x; }
    e.part[2 * bid] = s0; e.part[2 * bid + 1] = s1;
    unsigned t;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(e.gticket + g) : "memory");
    flag = t == gs - 1;
  }
  __syncthreads();
  if (!flag) return;
  if (warp != 0) return;
  // group finisher (one warp): slots of group g in order
  double2 p0 = make_double2(0, 0), p1 = make_double2(0, 0);
  if (lane < (int)gs) { p0 = __ldcg(e.part + 2 * (g * 32 + lane)); p1 = __ldcg(e.part + 2 * (g * 32 + lane) + 1); }
  p0 = warp_sum2(p0);
  p1 = warp_sum2(p1);
  unsigned last = 0;
  if (lane == 0) {
    e.gpart[2 * g] = p0; e.gpart[2 * g + 1] = p1;
    e.gticket[g] = 0;
    unsigned t;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(e.ticket) : "memory");
    last = t == ng - 1;
  }
  last = __shfl_sync(~0u, last, 0);
  if (!last) return;
  double2 q0 = make_double2(0, 0), q1 = make_double2(0, 0);
  for (unsigned b = lane; b < ng; b += 32) {
    const double2 u0 = __ldcg(e.gpart + 2 * b), u1 = __ldcg(e.gpart + 2 * b + 1);
    q0.x += u0.x; q0.y += u0.y; q1.x += u1.x;
  }
  q0 = warp_sum2(q0);
  q1 = warp_sum2(q1);
  if (lane == 0) { e.result[0] = q0; e.result[1] = q1; *e.ticket = 0; }
}

__device__ __forceinline__ C shfl_up1(C v) {
  C r; r.x = __shfl_up_sync(0xffffffffu, v.x, 1); r.y = __shfl_up_sync(0xffffffffu, v.y, 1); return r;
}
__device__ __forceinline__ C shfl_dn1(C v) {
  C r; r.x = __shfl_down_sync(0xffffffffu, v.x, 1); r.y = __shfl_down_sync(0xffffffffu, v.y, 1); return r;
}

// V8: V6 with x±1 from warp shuffles (lanes 0 / 31 load)
template <int ZC>
__global__ void __launch_bounds__(256) v8_march_shfl(const C* __restrict__ x, C* __restrict__ y, int nx, int ny,
                                                     int nz, Co k) {
  const int lane = threadIdx.x & 31;
  const int ix = blockIdx.x * 32 + lane;
  const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int zb = blockIdx.z * ZC;
  if (iy >= ny) return;                       // whole warps only (rows)
  const bool in = ix < nx;
  const int cx = in ? ix : nx - 1;
  const int plane = nx * ny;
  const C zero = czero<C>();
  const bool hxm = ix > 0, hxp = ix < nx - 1, hym = iy > 0, hyp = iy < ny - 1;
  const C* xp = x + (int64_t)zb * plane + cx + nx * iy;
  C* yp = y + (int64_t)zb * plane + cx + nx * iy;
  C below = zb > 0 ? xp[-plane] : zero;
  C cur = xp[0];
#pragma unroll
  for (int j = 0; j < ZC; ++j) {
    const int z = zb + j;
    if (z >= nz) break;
    const C above = z < nz - 1 ? xp[plane] : zero;
    const C ym = hym ? xp[-nx] : zero;
    const C yq = hyp ? xp[nx] : zero;
    C xm = shfl_up1(cur), xq = shfl_dn1(cur);
    if (lane == 0) xm = hxm ? xp[-1] : zero;
    if (lane == 31) xq = hxp ? xp[1] : zero;
    if (!hxm) xm = zero;
    if (!hxp) xq = zero;
    C acc = zero;
    mac(acc, k.oz, below);
    mac(acc, k.oy, ym);
    mac(acc, k.ox, xm);
    mac(acc, k.d, cur);
    mac(acc, k.ox, xq);
    mac(acc, k.oy, yq);
    mac(acc, k.oz, above);
    if (in) yp[0] = acc;
    below = cur;
    cur = above;
    xp += plane;
    yp += plane;
  }
}

// reference kernels: copy (y = x) and read-only (sum x into one slot per CTA)
__global__ void __launch_bounds__(256) k_copy(const C* __restrict__ x, C* __restrict__ y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) y[i] = __ldg(x + i);
}
__global__ void __launch_bounds__(256) k_read(const C* __restrict__ x, C* __restrict__ y, int64_t n) {
  C a = czero<C>();
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) a = cadd(a, __ldg(x + i));
  if (a.x == 12345.678) y[0] = a;
}
__global__ void __launch_bounds__(256) k_write(C* __restrict__ y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) y[i] = czero<C>();
}

#define CKE(x)                                                                  \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e_), __LINE__); exit(1); } \
  } while (0)

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  const int N = argc > 1 ? atoi(argv[1]) : 128;
  const int nx = N, ny = N, nz = N;
  const int64_t n = (int64_t)nx * ny * nz;
  std::vector<C> hx(n);
  uint64_t s = 12345;
  for (int64_t i = 0; i < n; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    hx[i].x = ((s >> 11) * (1.0 / 9007199254740992.0)) - 0.5;
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    hx[i].y = ((s >> 11) * (1.0 / 9007199254740992.0)) - 0.5;
  }
  C *x, *y, *yref, *flush;
  CKE(cudaMalloc(&x, n * sizeof(C)));
  CKE(cudaMalloc(&y, n * sizeof(C)));
  CKE(cudaMalloc(&yref, n * sizeof(C)));
  const size_t fbytes = 512ull << 20;
  CKE(cudaMalloc(&flush, fbytes));
  CKE(cudaMemcpy(x, hx.data(), n * sizeof(C), cudaMemcpyHostToDevice));
  const double kk = 25.0 / 4096.0;
  Co k{make_double2(6 - kk, -0.5 * kk), make_double2(-1, 0), make_double2(-1, 0), make_double2(-1, 0)};
  dim3 g3((nx + 31) / 32, (ny + 7) / 8, nz);
  v3_point<<<g3, 256>>>(x, yref, nx, ny, nz, k);
  CKE(cudaDeviceSynchronize());
  if (argc > 2) {   // profiling mode: a few warm launches of the main candidates
    dim3 g0((nx + 31) / 32, (ny + 7) / 8, (nz + 3) / 4);
    const size_t smb = 128 + (size_t)4 * 6 * nx * sizeof(C);
    cudaFuncSetAttribute(v5_bulk<4, 8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    for (int r = 0; r < 3; ++r) {
      v0_march<<<g0, 256>>>(x, y, nx, ny, nz, 4, k);
      v3_point<<<g3, 256>>>(x, y, nx, ny, nz, k);
      k_copy<<<296, 256>>>(x, y, n);
      v5_bulk<4, 8, 4><<<dim3(ny / 4, nz / 8), 256, smb>>>(x, y, nx, ny, nz, k);
    }
    CKE(cudaDeviceSynchronize());
    return 0;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  EpiOut eo;
  CKE(cudaMalloc(&eo.part, 2 * sizeof(double2) * 1 << 16));
  CKE(cudaMalloc(&eo.ticket, sizeof(unsigned)));
  CKE(cudaMemset(eo.ticket, 0, sizeof(unsigned)));
  CKE(cudaMalloc(&eo.result, 2 * sizeof(double2)));
  EpiOut2 eo2;
  CKE(cudaMalloc(&eo2.part, sizeof(double2) * 2 * 65536));
  CKE(cudaMalloc(&eo2.gpart, sizeof(double2) * 2 * 4096));
  CKE(cudaMalloc(&eo2.gticket, sizeof(unsigned) * 4096));
  CKE(cudaMemset(eo2.gticket, 0, sizeof(unsigned) * 4096));
  eo2.ticket = eo.ticket;
  eo2.result = eo.result;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = 2.0 * n * sizeof(C);
  auto bench = [&](const char* name, auto launch, bool flushl2) {
    CKE(cudaMemset(y, 0, n * sizeof(C)));
    launch();
    CKE(cudaGetLastError());
    CKE(cudaDeviceSynchronize());
    std::vector<C> a(n), b(n);
    CKE(cudaMemcpy(a.data(), y, n * sizeof(C), cudaMemcpyDeviceToHost));
    CKE(cudaMemcpy(b.data(), yref, n * sizeof(C), cudaMemcpyDeviceToHost));
    const bool same = memcmp(a.data(), b.data(), n * sizeof(C)) == 0;
    std::vector<float> ts;
    const int inner = flushl2 ? 1 : 20;   // warm: 20 back-to-back launches per sample (graph-replay-like)
    for (int r = 0; r < 30; ++r) {
      if (flushl2) CKE(cudaMemsetAsync(flush, r, fbytes));
      cudaEventRecord(e0);
      for (int q = 0; q < inner; ++q) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms * 1000.f / inner);
    }
    std::sort(ts.begin(), ts.end());
    printf("%-28s %s best %7.2f us  med %7.2f us  %6.0f GB/s (med)%s\n", name, flushl2 ? "cold" : "warm", ts[0],
           ts[ts.size() / 2], bytes / (ts[ts.size() / 2] * 1e-6) / 1e9, same ? "" : "  MISMATCH");
  };
  for (int fl = 1; fl >= 0; --fl) {
    bench("v3 point", [&] { v3_point<<<g3, 256>>>(x, y, nx, ny, nz, k); }, fl);
    for (int zc : {4, 8, 16}) {
      char nm[64];
      snprintf(nm, sizeof nm, "v0 march zc=%d", zc);
      dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + zc - 1) / zc);
      bench(nm, [&] { v0_march<<<g, 256>>>(x, y, nx, ny, nz, zc, k); }, fl);
    }
#define V1(ZC)                                                                                        \
  {                                                                                                   \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                         \
    bench("v1 march_shfl zc=" #ZC, [&] { v1_march_shfl<ZC><<<g, 256>>>(x, y, nx, ny, nz, k); }, fl); \
  }
    V1(4) V1(8) V1(16) V1(32)
#define V2(ZC, S)                                                                                        \
  {                                                                                                      \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                            \
    bench("v2 smem zc=" #ZC " S=" #S, [&] { v2_smem<ZC, S><<<g, 256>>>(x, y, nx, ny, nz, k); }, fl); \
  }
    V2(8, 4) V2(16, 4) V2(16, 6) V2(32, 4) V2(32, 6)
#define V5(TY, ZC, S)                                                                                    \
  {                                                                                                      \
    dim3 g((ny + TY - 1) / TY, (nz + ZC - 1) / ZC);                                                      \
    const size_t smb = 128 + (size_t)S * (TY + 2) * nx * sizeof(C);                                      \
    cudaFuncSetAttribute(v5_bulk<TY, ZC, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);     \
    bench("v5 bulk TY=" #TY " zc=" #ZC " S=" #S, [&] { v5_bulk<TY, ZC, S><<<g, 256, smb>>>(x, y, nx, ny, nz, k); }, fl); \
  }
    V5(2, 8, 4) V5(2, 16, 4) V5(4, 8, 4) V5(4, 16, 4) V5(4, 16, 5) V5(8, 8, 4) V5(8, 16, 4) V5(8, 8, 5) V5(4, 32, 4)
#define V4(ZC)                                                                                    \
  {                                                                                               \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                     \
    bench("v4 march2 zc=" #ZC, [&] { v4_march2<ZC><<<g, 128>>>(x, y, nx, ny, nz, k); }, fl); \
  }
    V4(4) V4(8) V4(16)
  }
  v3f_point<<<g3, 256>>>(x, yref, nx, ny, nz, k);   // FMA-accumulated reference from here on
  CKE(cudaDeviceSynchronize());
  for (int fl = 1; fl >= 0; --fl) {
    bench("v3f point (fma)", [&] { v3f_point<<<g3, 256>>>(x, y, nx, ny, nz, k); }, fl);
#define V6(ZC)                                                                                    \
  {                                                                                               \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                     \
    bench("v6 march fma zc=" #ZC, [&] { v6_march<ZC><<<g, 256>>>(x, y, nx, ny, nz, k); }, fl); \
  }
    V6(2) V6(4) V6(8) V6(16)
#define V7(ZC, R)                                                                                          \
  {                                                                                                        \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                              \
    bench("v7 rows R=" #R " zc=" #ZC, [&] { v7_march_rows<ZC, R><<<g, 256 / R>>>(x, y, nx, ny, nz, k); }, fl); \
  }
    V7(4, 2) V7(8, 2) V7(4, 4) V7(8, 4) V7(2, 2)
#define V8(ZC)                                                                                        \
  {                                                                                                   \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                         \
    bench("v8 shfl fma zc=" #ZC, [&] { v8_march_shfl<ZC><<<g, 256>>>(x, y, nx, ny, nz, k); }, fl); \
  }
    V8(4) V8(8)
#define V9(ZC, PD, MB)                                                                                     \
  {                                                                                                        \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                              \
    bench("v9 prefetch zc=" #ZC " pd=" #PD " minb=" #MB,                                                   \
          [&] { v9_prefetch<ZC, PD, MB><<<g, 256>>>(x, y, nx, ny, nz, k); }, fl);                          \
  }
    V9(8, 2, 1) V9(8, 3, 1) V9(8, 4, 1) V9(16, 3, 1) V9(16, 4, 1) V9(16, 6, 1) V9(32, 4, 1) V9(8, 3, 4) V9(16, 4, 4)
    V9(16, 4, 3) V9(32, 6, 3) V9(4, 2, 4) V9(4, 3, 4)
#define V10(ZC)                                                                                    \
  {                                                                                                \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                      \
    bench("v10 epi zc=" #ZC, [&] { v10_epi<ZC><<<g, 256>>>(x, y, nx, ny, nz, k, eo); }, fl);         \
  }
    V10(2) V10(4) V10(8)
#define V11(ZC, MB, W)                                                                                        \
  {                                                                                                           \
    int occ = 0;                                                                                              \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v11_persist<ZC, MB>, 256, 0);                        \
    const int grid = sms * occ * W;                                                                           \
    bench("v11 persist zc=" #ZC " minb=" #MB " waves=" #W,                                                    \
          [&] { v11_persist<ZC, MB><<<grid, 256>>>(x, y, nx, ny, nz, k, eo); }, fl);                          \
  }
    V11(2, 1, 1) V11(4, 1, 1) V11(8, 1, 1) V11(4, 3, 1) V11(4, 4, 1) V11(2, 4, 1) V11(4, 1, 2) V11(4, 4, 2)
#define V10R(ZC)                                                                                          \
  {                                                                                                       \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                             \
    bench("v10 epi release zc=" #ZC, [&] { v10_epi<ZC, true><<<g, 256>>>(x, y, nx, ny, nz, k, eo); }, fl); \
  }
    V10R(2) V10R(4) V10R(8)
#define V11R(ZC, MB)                                                                                          \
  {                                                                                                           \
    int occ = 0;                                                                                              \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v11_persist<ZC, MB, true>, 256, 0);                  \
    const int grid = sms * occ;                                                                               \
    bench("v11 persist release zc=" #ZC " minb=" #MB,                                                         \
          [&] { v11_persist<ZC, MB, true><<<grid, 256>>>(x, y, nx, ny, nz, k, eo); }, fl);                    \
  }
    V11R(4, 1) V11R(4, 4) V11R(8, 1)
    V11(4, 6, 1) V11(4, 8, 1) V11(8, 8, 1)
#define V12(ZC, M)                                                                                          \
  {                                                                                                         \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                               \
    bench("v12 parts mode=" #M " zc=" #ZC, [&] { v12_parts<ZC, M><<<g, 256>>>(x, y, nx, ny, nz, k, eo); }, fl); \
  }
    V12(4, 1) V12(4, 2) V12(8, 1) V12(8, 2)
#define V14(ZC)                                                                                          \
  {                                                                                                      \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                            \
    bench("v14 epi two-level zc=" #ZC, [&] { v14_epi2<ZC><<<g, 256>>>(x, y, nx, ny, nz, k, eo2); }, fl);  \
  }
    V14(2) V14(4) V14(8)
  }
  for (int fl = 1; fl >= 0; --fl) {
    bench("copy (cudaMemcpy d2d)", [&] { cudaMemcpyAsync(y, x, n * sizeof(C), cudaMemcpyDeviceToDevice); }, fl);
    for (int gm : {1, 2, 4, 8}) {
      char nm[64];
      snprintf(nm, sizeof nm, "k_copy grid=%dx148", gm);
      bench(nm, [&] { k_copy<<<148 * gm, 256>>>(x, y, n); }, fl);
    }
    bench("k_copy grid=n/256", [&] { k_copy<<<(int)((n + 255) / 256), 256>>>(x, y, n); }, fl);
    bench("k_read grid=8x148 (bytes/2)", [&] { k_read<<<148 * 8, 256>>>(x, y, n); }, fl);
    bench("k_write grid=8x148 (bytes/2)", [&] { k_write<<<148 * 8, 256>>>(y, n); }, fl);
  }
  return 0;
}
