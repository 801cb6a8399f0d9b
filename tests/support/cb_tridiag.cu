// Test-side user operator for ccg_set_matvec_callback (NOT part of the
// product): a complex tridiagonal matrix with constant diagonals, applied by
// a kernel the callback enqueues on the library's stream (graph-capturable).
#include <cuda_runtime.h>
#include <stdint.h>

struct Tri { double d[2], lo[2], up[2]; };

__global__ void tri_kernel(const double2* x, double2* y, int64_t n, int64_t row0, int64_t nloc, double2 d,
                           double2 lo, double2 up) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nloc) return;
  const int64_t g = row0 + i;
  double2 acc = make_double2(d.x * x[g].x - d.y * x[g].y, d.x * x[g].y + d.y * x[g].x);
  if (g > 0) { acc.x += lo.x * x[g - 1].x - lo.y * x[g - 1].y; acc.y += lo.x * x[g - 1].y + lo.y * x[g - 1].x; }
  if (g < n - 1) { acc.x += up.x * x[g + 1].x - up.y * x[g + 1].y; acc.y += up.x * x[g + 1].y + up.y * x[g + 1].x; }
  y[i] = acc;
}

extern "C" int cb_tridiag(void* user, int op, const void* x, void* y, int64_t n, int64_t row0, int64_t nloc,
                          void* stream) {
  const Tri* t = static_cast<const Tri*>(user);
  double2 d = make_double2(t->d[0], t->d[1]), lo = make_double2(t->lo[0], t->lo[1]),
          up = make_double2(t->up[0], t->up[1]);
  if (op != 0) { double2 s = lo; lo = up; up = s; }          // Aᵀ: swap the off-diagonals
  if (op == 1) { d.y = -d.y; lo.y = -lo.y; up.y = -up.y; }   // Aᴴ: and conjugate
  const int nt = 256;
  tri_kernel<<<(unsigned)((nloc + nt - 1) / nt), nt, 0, (cudaStream_t)stream>>>(
      (const double2*)x, (double2*)y, n, row0, nloc, d, lo, up);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
