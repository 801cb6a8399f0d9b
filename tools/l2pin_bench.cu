// l2pin_bench.cu — standalone microbenchmark: does marking a fraction of a
// dense c128 matrix L2::evict_last (createpolicy + ld.global.L2::cache_hint)
// keep it resident across repeated GEMVs, when the matrix is ~2x the L2?
// Development tool, not part of libccg.so.  Config 2 shape (n = 4096, c128,
// 256 MiB).  Rows with ((i >> 3) & 63) < q are loaded with an evict_last
// policy, the rest with ld.global.cs (evict-first); between variants the
// pinned lines are demoted with applypriority.global.L2::evict_normal.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        tools/l2pin_bench.cu -o /tmp/l2pin_bench
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CKE(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ unsigned long long pol_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld_keep(const double2* a, unsigned long long p) {
  double2 v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(p));
  return v;
}

template <int UR>
__global__ void __launch_bounds__(256) gemv(const double2* __restrict__ A, const double2* __restrict__ x,
                                            double2* __restrict__ y, int n, int q, int rows_per_cta) {
  extern __shared__ double2 xs[];
  for (int t = threadIdx.x; t < n; t += 256) xs[t] = x[t];
  __syncthreads();
  const unsigned long long pol = pol_last();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = blockIdx.x * rows_per_cta, i1 = min(n, i0 + rows_per_cta);
  for (int i = i0 + warp; i < i1; i += 8) {
    const double2* a = A + (size_t)i * n;
    const bool keep = ((i >> 3) & 63) < q;
    double ax = 0, ay = 0;
    for (int k = lane; k < n; k += 32 * UR) {
      double2 v[UR];
      if (keep) {
#pragma unroll
        for (int u = 0; u < UR; ++u) v[u] = ld_keep(a + k + 32 * u, pol);
      } else {
#pragma unroll
        for (int u = 0; u < UR; ++u) v[u] = __ldcs(a + k + 32 * u);
      }
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const double2 xv = xs[k + 32 * u];
        ax = fma(v[u].x, xv.x, ax); ax = fma(-v[u].y, xv.y, ax);
        ay = fma(v[u].x, xv.y, ay); ay = fma(v[u].y, xv.x, ay);
      }
    }
    for (int o = 16; o; o >>= 1) { ax += __shfl_xor_sync(~0u, ax, o); ay += __shfl_xor_sync(~0u, ay, o); }
    if (lane == 0) y[i] = make_double2(ax, ay);
  }
}

__global__ void demote(const char* p, size_t bytes) {
  for (size_t o = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 128; o < bytes; o += (size_t)gridDim.x * blockDim.x * 128)
    asm volatile("applypriority.global.L2::evict_normal [%0], 128;" :: "l"(p + o));
}

__global__ void fill(double2* a, size_t m) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x)
    a[i] = make_double2(1e-3 * (double)(i % 977), -1e-3 * (double)(i % 613));
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 4096;
  const int reps = 40;
  int dev = 0, sms = 0;
  CKE(cudaSetDevice(dev));
  CKE(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaDeviceProp prop;
  CKE(cudaGetDeviceProperties(&prop, dev));
  printf("L2 %d B, persistingL2CacheMaxSize %d B, accessPolicyMaxWindowSize %d B\n", prop.l2CacheSize,
         prop.persistingL2CacheMaxSize, prop.accessPolicyMaxWindowSize);
  const size_t m = (size_t)n * n, bytes = m * sizeof(double2);
  double2 *A, *x, *y;
  CKE(cudaMalloc(&A, bytes));
  CKE(cudaMalloc(&x, n * sizeof(double2)));
  CKE(cudaMalloc(&y, n * sizeof(double2)));
  fill<<<sms * 8, 256>>>(A, m);
  fill<<<64, 256>>>(x, n);
  CKE(cudaFuncSetAttribute(gemv<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, n * 16));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int setaside = 0; setaside < 2; ++setaside) {
    CKE(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setaside ? prop.persistingL2CacheMaxSize : 0));
    for (int rpc : {8, 16, 28}) {
      const int grid = (n + rpc - 1) / rpc;
      for (int q : {0, 8, 16, 20, 24, 28, 32, 40}) {
        demote<<<sms * 4, 256>>>((const char*)A, bytes);
        std::vector<float> t(reps);
        for (int r = 0; r < reps; ++r) {
          cudaEventRecord(e0);
          gemv<8><<<grid, 256, n * 16>>>(A, x, y, n, q, rpc);
          cudaEventRecord(e1);
          CKE(cudaEventSynchronize(e1));
          cudaEventElapsedTime(&t[r], e0, e1);
        }
        CKE(cudaGetLastError());
        std::sort(t.begin() + 2, t.end());
        const float med = t[2 + (reps - 2) / 2];
        printf("setaside=%d rows/cta=%2d pin=%2d/64 (%5.1f MB)  first %7.1f us  median %7.1f us  %6.0f GB/s eff\n",
               setaside, rpc, q, bytes * q / 64.0 / 1e6, t[0] * 1e3, med * 1e3, bytes / (med * 1e-3) / 1e9);
      }
    }
  }
  demote<<<sms * 4, 256>>>((const char*)A, bytes);
  CKE(cudaDeviceSynchronize());
  return 0;
}
