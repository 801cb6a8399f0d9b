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
