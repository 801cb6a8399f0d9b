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

#define CKE(x)                                                                  \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e_), __LINE__); exit(1); } \
  } while (0)

int main(int argc, char** argv) {
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
    for (int r = 0; r < 30; ++r) {
      if (flushl2) CKE(cudaMemsetAsync(flush, r, fbytes));
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms * 1000.f);
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
#define V4(ZC)                                                                                    \
  {                                                                                               \
    dim3 g((nx + 31) / 32, (ny + 7) / 8, (nz + ZC - 1) / ZC);                                     \
    bench("v4 march2 zc=" #ZC, [&] { v4_march2<ZC><<<g, 128>>>(x, y, nx, ny, nz, k); }, fl); \
  }
    V4(4) V4(8) V4(16)
  }
  // copy roofline for reference: y = x
  bench("copy (cudaMemcpy d2d)", [&] { cudaMemcpyAsync(y, x, n * sizeof(C), cudaMemcpyDeviceToDevice); }, true);
  return 0;
}
