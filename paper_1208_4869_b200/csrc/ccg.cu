// ccg.cu — libccg.so: C-ABI (include/ccg.h), matvec engine dispatch, the
// per-method iteration schedules, CUDA-graph iteration loop and the NCCL
// row-sharded multi-GPU path.
//
// Paper mapping (PAPER.md = P:<line>):  matvec / cmatvec separated from the
// iteration (P:17, P:95 [§5]) -> ccg_set_matvec_* + the kernels of
// matvec.cuh; cgmodule's epsilon_err / maxit -> ccg_solve(tol, maxit);
// ddprecision.f90 single/double switch -> ccg_dtype.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/ccg.h"
#include "common.cuh"
#include "matvec.cuh"
#include "methods.cuh"
#include "comm.cuh"
#include "fft.cuh"
#include "cluster.cuh"
#include "gmres.cuh"

#include <complex>

using namespace ccg;

namespace {
thread_local std::string g_create_err;
}  // namespace

// ===========================================================================
// context
// ===========================================================================
enum { NLOCAL = 12, NFULL = 3 };
enum { OPK_NONE = 0, OPK_DENSE = 1, OPK_CSR = 2, OPK_STENCIL = 3, OPK_TOEPLITZ = 4, OPK_CALLBACK = 5 };
enum { GEMV_SPLIT = 0, GEMV_BULK = 1, GEMV_ROWS = 2, GEMV_COLS = 3 };

struct ccg_ctx {
  int dtype = 0;
  int64_t n = 0, nloc = 0, row0 = 0;   // vector slice of this rank (whole vector when rep)
  int64_t mnloc = 0, mrow0 = 0;         // operator rows of this rank (= nloc, row0 unless rep)
  bool rep = false;                     // replicated-vector mode (SURVEY §8(f) NEXT-2 ii)
  void* rep_tmp = nullptr;              // n: product rows gathered from every rank
  void* rep_parts = nullptr;            // world × n: Aᴴ partials of every rank
  int world = 1, rank = 0, device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  size_t esz = 8;  // bytes per complex
  // operator
  int opk = OPK_NONE;
  const void* A = nullptr;
  int64_t lda = 0;
  uint32_t flags = 0;
  const int32_t* rowptr = nullptr;
  const int32_t* colind = nullptr;
  const void* vals = nullptr;
  int64_t nnz = 0, halo = 0;
  int32_t* csr_blocks = nullptr;  // CSR-stream row-block boundaries (device)
  int csr_nblocks = 0;
  int64_t* sell_off = nullptr;    // SELL-32 copy of the CSR operator (owned)
  int32_t* sell_width = nullptr;
  int32_t* sell_col = nullptr;
  void* sell_val = nullptr;
  int sell_grid[2] = {0, 0};
  int sell_one = 0, sell_waves = 1;   // SELL load schedule / grid waves (CCG_SELL_ONE, CCG_SELL_WAVES)
  // matrix-free 7-point stencil (ccg_set_matvec_stencil7)
  int snx = 0, sny = 0, snz = 0, sz0 = 0, snzl = 0, szc = 4;
  double2 scoef[4] = {};  // d, ox, oy, oz
  // FFT block-Toeplitz operator (ccg_set_matvec_toeplitz3)
  FftGeo geo = {};
  void* fftW = nullptr;   // padded work array X2·Y2·Z2
  void* fftK = nullptr;   // K̂ / (X2·Y2·Z2)
  void* fftTw = nullptr;  // exp(−2πi k/Lmax), k < Lmax/2
  int fft_lmax = 1;
  double2 tdiag = {};
  // user matvec callback (ccg_set_matvec_callback)
  ccg_matvec_fn cb_fn = nullptr;
  void* cb_user = nullptr;
  uint32_t cb_caps = 0;
  void* cb_out = nullptr;   // nloc output rows of the user's product
  // GMRES(m) workspace (gmres.cuh)
  int gm_m = 30;
  GmDev* gm_dev = nullptr;
  void* gm_V = nullptr;     // (m+1) × nloc basis
  size_t gm_V_bytes = 0;
  double2* gm_part = nullptr;
  unsigned* gm_ticket = nullptr;
  double2* gm_rank = nullptr;
  double2* gm_all = nullptr;
  int gm_grid = 1;
  int gm_fast = 1;   // unrolled multi-dot loads (CCG_GM_FAST=0 disables)
  int gm_vgrid = 1;  // one wave of gm_normalize / gm_xupdate
  // BiCGstab(ℓ) workspace: r̂₀..r̂_ℓ, û₀..û_ℓ as full-length buffers
  int bl_l = 2, bl_built = 0;
  void* bl_buf = nullptr;
  size_t bl_bytes = 0;
  // right Jacobi preconditioning (ccg_set_jacobi): d and 1/d over all n rows
  void* jac_d = nullptr;
  void* jac_dinv = nullptr;
  void* jac_tmp = nullptr;   // n: D⁻¹·(product input)
  bool jac_active = false;   // inside ccg_solve
  // whole-loop cluster kernel for small dense systems (cluster.cuh)
  bool cluster_ok = false;
  int cluster_size = 0;   // 0 = not yet chosen
  int cl_method = 0, cl_has_x0 = 0;
  bool vec_ok = true;
  bool bulk_ok = false;   // TMA bulk-copy GEMV usable (alignment / n multiple of a 4 KiB tile)
  int bulk_grid = 0;
  int gemv_mode = 0;      // GEMV_SPLIT (default) | GEMV_BULK | GEMV_ROWS (env CCG_GEMV)
  int split_W = 0, split_strips = 1, split_nrb = 1, nstage2_grid = 1, split_ur = 8;
  bool cols_ok = false;   // column-owner GEMV usable (vectorised layout, n % V == 0)
  int cols_strips = 1, cols_S = 1, dual_S = 1, cols_rg = 1;
  bool qmr_dual = true;   // QMR: A·p and Aᴴ·q in one pass over A (env CCG_QMR_DUAL=0 disables)
  void* npart = nullptr;  // [strips][nloc] partial row sums of the split / column-owner GEMV
  size_t npart_bytes = 0;
  // workspace
  State* st = nullptr;
  State* st_host = nullptr;  // pinned
  int* done_ring = nullptr;   // pinned: done-flag copies of the last two queued chunks
  cudaEvent_t done_ev[2] = {nullptr, nullptr};
  bool pipe = false;          // pipelined chunk launches (CCG_PIPELINE=1; off by default)
  double2* part = nullptr;
  size_t part_cap = 0;  // in double2
  unsigned* ticket = nullptr;
  double2* rank_sum = nullptr;
  double2* all_sums = nullptr;
  int* zero_gate = nullptr;
  void* loc[NLOCAL] = {};
  void* full[NFULL] = {};
  void* hpart = nullptr;
  size_t hpart_bytes = 0;
  void* wfull = nullptr;
  double* hist = nullptr;
  int hist_cap = 0;
  int hist_len = 0;
  void* stage_in = nullptr;  // pinned staging (host pointer I/O)
  size_t stage_bytes = 0;
  // comm
  Comm* comm = nullptr;  // NcclComm or LoopbackComm (world > 1)
  // graphs per method
  cudaGraphExec_t gexec[M_COUNT] = {};
  int64_t graph_launches_per_iter[M_COUNT] = {};
  // launch parameters
  int sm_count = 148;
  int gemv_grid = 0, ah_S = 1, ah_strips = 1, pass_grid = 0, stage2_grid = 0, spmv_grid = 0;
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;
  std::vector<int> ev_kind;
  double ms_a = 0, ms_ah = 0;
  int n_a = 0, n_ah = 0;
  int64_t launches = 0;
  bool capturing = false;
  bool pdl = true;        // programmatic dependent launch (env CCG_PDL=0 disables)
  std::string err;
};

// kernel launch, with the programmatic-dependent-launch attribute unless
// disabled (CCG_PDL=0): every launched kernel begins with pdl_gate()/pdl_wait()
template <typename... KArgs, typename... Args>
static void launch_k(ccg_ctx* c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args);

#define FAIL(c, code, msg)       \
  do {                           \
    (c)->err = (msg);            \
    return (code);               \
  } while (0)

#define CK(c, call)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      (c)->err = std::string(#call) + " (line " + std::to_string(__LINE__) + "): " + cudaGetErrorString(e_); \
      return CCG_E_CUDA;                                                                   \
    }                                                                                      \
  } while (0)

#define NK(c, call)                 \
  do {                              \
    int r_ = (call);                \
    if (r_ != 0) {                  \
      (c)->err = (c)->comm->err;    \
      return r_;                    \
    }                               \
  } while (0)

#define TRY(expr)            \
  do {                       \
    int rc_ = (expr);        \
    if (rc_ != CCG_OK) return rc_; \
  } while (0)

template <typename... KArgs, typename... Args>
static void launch_k(ccg_ctx* c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  if (!c->pdl) {
    kern<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) {
    fprintf(stderr, "libccg: launch failed (%s): grid %u,%u,%u block %u smem %zu\n", cudaGetErrorString(e), grid.x,
            grid.y, grid.z, block.x, smem);
  }
}

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static Red make_red(ccg_ctx* c) {
  Red r;
  r.part = c->part;
  r.ticket = c->ticket;
  r.rank_sum = c->rank_sum;
  r.fuse = (c->world == 1 || c->rep) ? 1 : 0;   // replicated vectors: reductions are local
  return r;
}

// ---------------------------------------------------------------------------
// timing events around matvec launches (kind 0 = A, 1 = AH)
// ---------------------------------------------------------------------------
static void tev_begin(ccg_ctx* c, int kind) {
  if (!c->timing) return;
  if (c->ev_used + 2 > c->ev.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->ev.push_back(e);
    }
  }
  cudaEventRecord(c->ev[c->ev_used], c->stream);
  c->ev_kind.push_back(kind);
}
static void tev_end(ccg_ctx* c) {
  if (!c->timing) return;
  cudaEventRecord(c->ev[c->ev_used + 1], c->stream);
  c->ev_used += 2;
}
static void tev_collect(ccg_ctx* c) {
  if (!c->timing) return;
  cudaStreamSynchronize(c->stream);
  for (size_t p = 0; p < c->ev_kind.size(); ++p) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[2 * p], c->ev[2 * p + 1]);
    if (c->ev_kind[p] == 0) { c->ms_a += ms; c->n_a++; } else { c->ms_ah += ms; c->n_ah++; }
  }
  c->ev_used = 0;
  c->ev_kind.clear();
}

// ===========================================================================
// Engine<T>: launches
// ===========================================================================
template <typename T>
struct Engine {
  using C = typename CT<T>::c;
  static constexpr int NT = 256;
  static constexpr int R = 8;
  static constexpr int UR = 8;
  static constexpr int LPR = 8;
  static constexpr int BR = 8;        // rows per group, bulk GEMV
  static constexpr int BSTAGES = 5;   // pipeline depth, bulk GEMV (5 x 36 KiB smem)
  static constexpr int SUR = 8;       // 16-byte loads in flight per lane, split GEMV
  static constexpr int SNNZ = 2048;   // nonzeros per CSR-stream block

  static C* L(ccg_ctx* c, int i) { return reinterpret_cast<C*>(c->loc[i]); }
  static C* F(ccg_ctx* c, int i) { return reinterpret_cast<C*>(c->full[i]); }
  static C* Fs(ccg_ctx* c, int i) { return reinterpret_cast<C*>(c->full[i]) + c->row0; }  // own slice

  static CommType ndt() { return sizeof(T) == 4 ? CT_F32 : CT_F64; }

  // -------------------- collectives --------------------
  static int allgather(ccg_ctx* c, int fi) {
    if (c->world == 1 || c->rep) return CCG_OK;   // replicated vectors are whole on every rank
    C* buf = F(c, fi);
    if (c->opk == OPK_CSR || c->opk == OPK_STENCIL) return halo_exchange(c, buf);
    // dense and FFT-Toeplitz: every rank needs the whole input vector
    NK(c, c->comm->allgather_inplace(buf, (size_t)c->nloc * 2, ndt(), c->stream));
    return CCG_OK;
  }
  static int halo_exchange(ccg_ctx* c, C* buf) {
    NK(c, c->comm->halo(buf, c->row0, c->nloc, c->halo, sizeof(C), ndt(), c->stream));
    return CCG_OK;
  }
  // scalar phase for world > 1: allgather this rank's K sums, sum in rank order
  template <class Fin>
  static int post(ccg_ctx* c, const int* gate) {
    constexpr int K = Fin::K;
    if constexpr (K > 0) {
      if (c->world > 1 && !c->rep) {
        NK(c, c->comm->allgather(c->rank_sum, c->all_sums, (size_t)K * 2, CT_F64, c->stream));
        launch_k(c, scalar_kernel<K, Fin>, 1, 1, 0, c->stream, c->all_sums, c->world, c->st, gate);
        c->launches++;
      }
    }
    return CCG_OK;
  }

  // -------------------- kernels --------------------
  template <class Op>
  static int pass(ccg_ctx* c, Op op, const int* gate) {
    // whole waves at this functor's own occupancy (register use differs
    // between phases: 32-48 registers => 5-8 CTAs per SM)
    static int occ = 0;
    if (occ == 0) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass_kernel<NT, Op>, NT, 0);
      occ = std::max(1, std::min(occ, 8));
    }
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((c->nloc + NT - 1) / NT, (int64_t)c->sm_count * occ));
    launch_k(c, pass_kernel<NT, Op>, grid, NT, 0, c->stream, op, c->nloc, make_red(c), c->st, gate);
    c->launches++;
    CK(c, cudaGetLastError());
    return post<Op>(c, gate);
  }

  // a K = 0 elementwise pass over `count` elements (the whole vector)
  template <class Op>
  static int pass_count(ccg_ctx* c, Op op, int64_t count, const int* gate) {
    static_assert(Op::K == 0, "pass_count: no reduction");
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((count + NT - 1) / NT, (int64_t)c->sm_count * 8));
    launch_k(c, pass_kernel<NT, Op>, grid, NT, 0, c->stream, op, count, make_red(c), c->st, gate);
    c->launches++;
    CK(c, cudaGetLastError());
    return CCG_OK;
  }

  // CSR SpMV: CSR-stream blocks (default) or LPR lanes per row (CCG_SPMV=lanes)
  template <bool CONJ, class Epi>
  static void spmv(ccg_ctx* c, const C* x, Epi epi, const int* gate) {
    const C* vals = reinterpret_cast<const C*>(c->vals);
    if (c->sell_col) {
      auto k = c->sell_one ? spmv_sell_kernel<T, NT, CONJ, true, Epi> : spmv_sell_kernel<T, NT, CONJ, false, Epi>;
      launch_k(c, k, c->sell_grid[c->sell_one], NT, 0, c->stream,
          c->sell_off, c->sell_width, c->sell_col, reinterpret_cast<const C*>(c->sell_val), x, c->mnloc, epi,
          make_red(c), c->st, gate);
    }
    else if (c->csr_blocks)
      launch_k(c, spmv_stream_kernel<T, NT, SNNZ, CONJ, Epi>, c->spmv_grid, NT, 0, c->stream, 
          c->rowptr, c->colind, vals, x, c->csr_blocks, c->csr_nblocks, epi, make_red(c), c->st, gate);
    else
      launch_k(c, spmv_csr_kernel<T, LPR, NT, CONJ, Epi>, c->spmv_grid, NT, 0, c->stream, 
          c->rowptr, c->colind, vals, x, c->mnloc, epi, make_red(c), c->st, gate);
  }

  // matrix-free stencil; conj => Aᴴ (= the stencil with conjugated
  // coefficients, A being complex symmetric)
  template <class Epi>
  static void stencil(ccg_ctx* c, const C* xfull, bool conj, Epi epi, const int* gate) {
    C k[4];
    for (int i = 0; i < 4; ++i) {
      k[i].x = (T)c->scoef[i].x;
      k[i].y = (T)(conj ? -c->scoef[i].y : c->scoef[i].y);
    }
    dim3 g((c->snx + 31) / 32, (c->sny + 7) / 8, (c->snzl + c->szc - 1) / c->szc);
    launch_k(c, stencil7_kernel<T, Epi>, g, 256, 0, c->stream, xfull, c->snx, c->sny, c->snz, c->sz0, c->snzl, c->szc,
                                                       k[0], k[1], k[2], k[3], epi, make_red(c), c->st, gate);
  }

  // FFT block-Toeplitz product (fft.cuh); op: 0 = A, 1 = Aᴴ, 2 = Aᵀ.  Every
  // rank transforms the whole (gathered) vector and keeps its own rows.
  template <class Epi>
  static void toeplitz(ccg_ctx* c, const C* xfull, int op, Epi epi, const int* gate) {
    const FftGeo& g = c->geo;
    C* W = reinterpret_cast<C*>(c->fftW);
    const C* Kh = reinterpret_cast<const C*>(c->fftK);
    const C* tw = reinterpret_cast<const C*>(c->fftTw);
    const int L = c->fft_lmax;
    const size_t smx = (size_t)g.tx * g.X2 * sizeof(C);
    const size_t smy = (size_t)g.tyz * g.Y2 * sizeof(C);
    const size_t smz = (size_t)g.tyz * g.Z2 * sizeof(C);
    const int gx = (g.ny * g.nz + g.tx - 1) / g.tx;
    // threads per CTA: one per butterfly of its lines (a multiple of 32, ≤ 256)
    auto bt = [](int lines, int len) { return std::max(32, std::min(256, ((lines * len / 2 + 31) / 32) * 32)); };
    const int btx = bt(g.tx, g.X2), bty = bt(g.tyz, g.Y2), btz = bt(g.tyz, g.Z2);
    if (op == 1)
      launch_k(c, fft_fwd_x<T, true>, gx, btx, smx, c->stream, xfull, W, g, tw, L / g.X2, gate);
    else
      launch_k(c, fft_fwd_x<T, false>, gx, btx, smx, c->stream, xfull, W, g, tw, L / g.X2, gate);
    launch_k(c, fft_fwd_y<T>, dim3(g.X2 / g.tyz, g.nz), bty, smy, c->stream, W, g, tw, L / g.Y2, gate);
    if (op == 0)
      launch_k(c, fft_z_mul<T, false>, dim3(g.X2 / g.tyz, g.Y2), btz, smz, c->stream, W, Kh, g, tw, L / g.Z2, gate);
    else
      launch_k(c, fft_z_mul<T, true>, dim3(g.X2 / g.tyz, g.Y2), btz, smz, c->stream, W, Kh, g, tw, L / g.Z2, gate);
    launch_k(c, fft_inv_y<T>, dim3(g.X2 / g.tyz, g.nz), bty, smy, c->stream, W, g, tw, L / g.Y2, gate);
    C d;
    d.x = (T)c->tdiag.x;
    d.y = (T)(op == 1 ? -c->tdiag.y : c->tdiag.y);
    if (op == 1)
      launch_k(c, fft_inv_x<T, true, Epi>, gx, 256, smx, c->stream, W, xfull, g, tw, L / g.X2, d, c->row0, c->nloc, epi,
                                                            make_red(c), c->st, gate);
    else
      launch_k(c, fft_inv_x<T, false, Epi>, gx, 256, smx, c->stream, W, xfull, g, tw, L / g.X2, d, c->row0, c->nloc, epi,
                                                             make_red(c), c->st, gate);
    c->launches += 4;
  }

  // the user's product (ccg_set_matvec_callback) into cb_out, then the
  // method's epilogue as one fused pass over it
  template <class Epi>
  static int user_product(ccg_ctx* c, int op, const C* xfull, Epi epi, const int* gate) {
    C* out = c->rep ? reinterpret_cast<C*>(c->rep_tmp) : reinterpret_cast<C*>(c->cb_out);
    tev_begin(c, op == CCG_OP_A ? 0 : 1);
    const int rc = c->cb_fn(c->cb_user, op, xfull, c->rep ? out + c->mrow0 : out, c->n, c->mrow0, c->mnloc,
                            c->stream);
    tev_end(c);
    if (rc != 0) FAIL(c, CCG_E_USER, "user matvec callback returned " + std::to_string(rc));
    CK(c, cudaGetLastError());
    if (c->rep) NK(c, c->comm->allgather_inplace(out, (size_t)c->mnloc * 2, ndt(), c->stream));
    EpiPass<C, Epi> ep{epi, out};
    return pass(c, ep, gate);
  }

  // replicated vectors: this rank's product rows (Store into rep_tmp at mrow0),
  // allgathered, then the method epilogue as one pass over the whole vector
  template <class Epi>
  static int rep_finish_rows(ccg_ctx* c, Epi epi, const int* gate) {
    C* tmp = reinterpret_cast<C*>(c->rep_tmp);
    NK(c, c->comm->allgather_inplace(tmp, (size_t)c->mnloc * 2, ndt(), c->stream));
    EpiPass<C, Epi> ep{epi, tmp};
    return pass(c, ep, gate);
  }

  // y_local = A · xfull (full-length buffer, own slice + gathered/halo parts)
  template <class Epi>
  static int matvec_a(ccg_ctx* c, const C* xfull, Epi epi, const int* gate) {
    if (c->jac_active) {   // B·v = A(D⁻¹v): scale the (whole) input first
      C* tmp = reinterpret_cast<C*>(c->jac_tmp);
      TRY(pass_count(c, JacScale<T>{xfull, reinterpret_cast<const C*>(c->jac_dinv), tmp}, c->n, gate));
      xfull = tmp;
    }
    if (c->opk == OPK_CALLBACK) return user_product(c, CCG_OP_A, xfull, epi, gate);
    if (c->rep && c->opk != OPK_TOEPLITZ) {
      TRY(matvec_rows(c, xfull, Store<T>{reinterpret_cast<C*>(c->rep_tmp) + c->mrow0}, gate));
      return rep_finish_rows(c, epi, gate);
    }
    return matvec_rows(c, xfull, epi, gate);
  }

  // this rank's rows of A·x (all operators), epilogue per row
  template <class Epi>
  static int matvec_rows(ccg_ctx* c, const C* xfull, Epi epi, const int* gate) {
    tev_begin(c, 0);
    if (c->opk == OPK_TOEPLITZ) {
      toeplitz(c, xfull, 0, epi, gate);
    } else if (c->opk == OPK_STENCIL) {
      stencil(c, xfull, false, epi, gate);
    } else if (c->opk == OPK_DENSE && c->gemv_mode == GEMV_SPLIT) {
      const C* A = reinterpret_cast<const C*>(c->A);
      C* part = reinterpret_cast<C*>(c->npart);
      dim3 g(c->split_strips, c->split_nrb);
      const size_t smem = (size_t)c->split_W * sizeof(C);
      if (c->split_strips == 1) {
        if (c->vec_ok)
          launch_k(c, gemv_n_split<T, NT, SUR, true, true, Epi>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, epi, make_red(c), c->st, gate);
        else
          launch_k(c, gemv_n_split<T, NT, SUR, false, true, Epi>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, epi, make_red(c), c->st, gate);
      } else {
        Store<T> none{nullptr};
        if (c->vec_ok && c->split_ur == 16)
          launch_k(c, gemv_n_split<T, NT, 16, true, false, Store<T>>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, none, make_red(c), c->st, gate);
        else if (c->vec_ok && c->split_ur == 4)
          launch_k(c, gemv_n_split<T, NT, 4, true, false, Store<T>>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, none, make_red(c), c->st, gate);
        else if (c->vec_ok)
          launch_k(c, gemv_n_split<T, NT, SUR, true, false, Store<T>>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, none, make_red(c), c->st, gate);
        else
          launch_k(c, gemv_n_split<T, NT, SUR, false, false, Store<T>>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, none, make_red(c), c->st, gate);
        c->launches++;
        CK(c, cudaGetLastError());
        launch_k(c, gemv_h_stage2<T, NT, Epi>, c->nstage2_grid, NT, 0, c->stream, part, c->split_strips, c->mnloc, 0,
                                                                          c->mnloc, epi, make_red(c), c->st, gate);
      }
    } else if (c->opk == OPK_DENSE && c->gemv_mode == GEMV_COLS && c->cols_ok) {
      C* part = reinterpret_cast<C*>(c->npart);
      if (c->cols_rg == 4)
        launch_k(c, gemv_cols<T, NT, true, false, false, 4>, dim3(c->cols_strips, c->cols_S), NT, 0, c->stream, 
            reinterpret_cast<const C*>(c->A), c->lda, xfull, nullptr, c->mnloc, c->n, part, nullptr, gate);
      else
        launch_k(c, gemv_cols<T, NT, true, false, false, 1>, dim3(c->cols_strips, c->cols_S), NT, 0, c->stream, 
            reinterpret_cast<const C*>(c->A), c->lda, xfull, nullptr, c->mnloc, c->n, part, nullptr, gate);
      c->launches++;
      CK(c, cudaGetLastError());
      launch_k(c, gemv_h_stage2<T, NT, Epi>, c->nstage2_grid, NT, 0, c->stream, part, c->cols_strips, c->mnloc, 0, c->mnloc,
                                                                        epi, make_red(c), c->st, gate);
    } else if (c->opk == OPK_DENSE && c->gemv_mode == GEMV_BULK && c->bulk_ok) {
      constexpr size_t smem = bulk_smem_bytes<BR, BSTAGES>();
      auto kern = gemv_n_bulk<T, BR, BSTAGES, Epi>;
      static bool attr_set = false;  // per instantiation
      if (!attr_set) {
        CK(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set = true;
      }
      launch_k(c, kern, c->bulk_grid, BULK_NT, smem, c->stream, reinterpret_cast<const C*>(c->A), c->lda, xfull, c->n,
                                                       c->mnloc, epi, make_red(c), c->st, gate);
    } else if (c->opk == OPK_DENSE) {
      const C* A = reinterpret_cast<const C*>(c->A);
      if (c->vec_ok)
        launch_k(c, gemv_n_kernel<T, R, NT, true, Epi>, c->gemv_grid, NT, 0, c->stream, 
            A, c->lda, xfull, c->n, c->mnloc, epi, make_red(c), c->st, gate);
      else
        launch_k(c, gemv_n_kernel<T, R, NT, false, Epi>, c->gemv_grid, NT, 0, c->stream, 
            A, c->lda, xfull, c->n, c->mnloc, epi, make_red(c), c->st, gate);
    } else {
      spmv<false>(c, xfull, epi, gate);
    }
    c->launches++;
    tev_end(c);
    CK(c, cudaGetLastError());
    return post<Epi>(c, gate);
  }

  // y_local = op(A) · x_local, op = Aᴴ (conj) or Aᵀ.  With replicated vectors
  // x_local is the whole vector: complex-symmetric operators compute their own
  // rows, the dense product this rank's full-length partial, summed over ranks
  // in rank order inside the epilogue pass.
  template <class Epi>
  static int matvec_h(ccg_ctx* c, const C* xloc, bool conj, Epi epi, const int* gate) {
    if (c->jac_active) {   // Bᴴv = conj(D⁻¹)(Aᴴv), Bᵀv = D⁻¹(Aᵀv): scale inside the epilogue
      JacEpi<T, Epi> je{epi, reinterpret_cast<const C*>(c->jac_dinv) + c->row0, conj ? 1 : 0};
      return matvec_h_impl(c, xloc, conj, je, gate);
    }
    return matvec_h_impl(c, xloc, conj, epi, gate);
  }
  template <class Epi>
  static int matvec_h_impl(ccg_ctx* c, const C* xloc, bool conj, Epi epi, const int* gate) {
    const bool gathered_in = c->world > 1 && !c->rep;   // the input needs gathering first
    if (c->opk == OPK_CALLBACK) {
      const C* xin = xloc;
      if (gathered_in) {
        CK(c, cudaMemcpyAsync(Fs(c, 2), xloc, c->nloc * sizeof(C), cudaMemcpyDeviceToDevice, c->stream));
        TRY(allgather(c, 2));
        xin = F(c, 2);
      }
      return user_product(c, conj ? CCG_OP_AH : CCG_OP_AT, xin, epi, gate);
    }
    if (c->opk == OPK_TOEPLITZ) {
      const C* xin = xloc;
      if (gathered_in) {
        CK(c, cudaMemcpyAsync(Fs(c, 2), xloc, c->nloc * sizeof(C), cudaMemcpyDeviceToDevice, c->stream));
        TRY(allgather(c, 2));
        xin = F(c, 2);
      }
      tev_begin(c, 1);
      toeplitz(c, xin, conj ? 1 : 2, epi, gate);
      c->launches++;
      tev_end(c);
      CK(c, cudaGetLastError());
      return post<Epi>(c, gate);
    }
    if (c->opk == OPK_STENCIL || c->opk == OPK_CSR) {
      // complex-symmetric operator: Aᵀ = A, Aᴴx = conj(A conj x) (the stencil
      // conjugates its coefficients); its own rows from the whole input
      const C* xin = xloc;
      if (gathered_in) {
        CK(c, cudaMemcpyAsync(Fs(c, 2), xloc, c->nloc * sizeof(C), cudaMemcpyDeviceToDevice, c->stream));
        TRY(allgather(c, 2));
        xin = F(c, 2);
      }
      auto launch = [&](auto e) {
        if (c->opk == OPK_STENCIL) stencil(c, xin, conj, e, gate);
        else if (conj) spmv<true>(c, xin, e, gate);
        else spmv<false>(c, xin, e, gate);
      };
      tev_begin(c, 1);
      if (c->rep) launch(Store<T>{reinterpret_cast<C*>(c->rep_tmp) + c->mrow0});
      else launch(epi);
      c->launches++;
      tev_end(c);
      CK(c, cudaGetLastError());
      if (c->rep) return rep_finish_rows(c, epi, gate);
      return post<Epi>(c, gate);
    }
    const C* A = reinterpret_cast<const C*>(c->A);
    C* part = reinterpret_cast<C*>(c->hpart);
    const C* xr = c->rep ? xloc + c->mrow0 : xloc;   // the x entries of this rank's rows
    dim3 g1(c->ah_strips, c->ah_S);
    tev_begin(c, 1);
    if (c->vec_ok) {
      if (conj)
        launch_k(c, gemv_h_stage1<T, true, NT, UR, true>, g1, NT, 0, c->stream, A, c->lda, xr, c->mnloc, c->n, part, gate);
      else
        launch_k(c, gemv_h_stage1<T, false, NT, UR, true>, g1, NT, 0, c->stream, A, c->lda, xr, c->mnloc, c->n, part, gate);
    } else {
      if (conj)
        launch_k(c, gemv_h_stage1<T, true, NT, UR, false>, g1, NT, 0, c->stream, A, c->lda, xr, c->mnloc, c->n, part, gate);
      else
        launch_k(c, gemv_h_stage1<T, false, NT, UR, false>, g1, NT, 0, c->stream, A, c->lda, xr, c->mnloc, c->n, part, gate);
    }
    c->launches++;
    CK(c, cudaGetLastError());
    if (c->world == 1) {
      launch_k(c, gemv_h_stage2<T, NT, Epi>, c->stage2_grid, NT, 0, c->stream, part, c->ah_S, c->n, 0, c->n, epi,
                                                                       make_red(c), c->st, gate);
      c->launches++;
      tev_end(c);
      CK(c, cudaGetLastError());
      return CCG_OK;
    }
    // multi GPU: full-length partial of this rank
    C* wf = c->rep ? reinterpret_cast<C*>(c->rep_tmp) : reinterpret_cast<C*>(c->wfull);
    Store<T> stv{wf};
    launch_k(c, gemv_h_stage2<T, NT, Store<T>>, c->stage2_grid, NT, 0, c->stream, part, c->ah_S, c->n, 0, c->n, stv,
                                                                         make_red(c), c->st, gate);
    c->launches++;
    tev_end(c);
    CK(c, cudaGetLastError());
    if (c->rep) {
      // every rank's partial, summed in rank order inside the epilogue pass
      C* parts = reinterpret_cast<C*>(c->rep_parts);
      NK(c, c->comm->allgather(wf, parts, (size_t)c->n * 2, ndt(), c->stream));
      EpiPassSum<C, Epi> ep{epi, parts, c->world, c->n};
      return pass(c, ep, gate);
    }
    C* wl = L(c, NLOCAL - 1);   // row-sharded: reduce-scatter -> epilogue pass
    NK(c, c->comm->reduce_scatter(c->wfull, wl, (size_t)c->nloc * 2, ndt(), c->stream));
    EpiPass<C, Epi> ep{epi, wl};
    return pass(c, ep, gate);
  }

  // p̃ = A·p (epilogue ea) and w = Aᴴ·q (epilogue eh) in ONE pass over A
  // (gemv_cols<DO_N, DO_H>).  ea's scalar step runs
  // before eh's epilogue (QMR: ε, β before w̃ = Aᴴq − conj(β)w).
  template <class EpiA, class EpiH>
  static int matvec_dual(ccg_ctx* c, const C* pfull, const C* qloc, EpiA ea, EpiH eh, const int* gate) {
    const C* A = reinterpret_cast<const C*>(c->A);
    C* np = reinterpret_cast<C*>(c->npart);
    C* hp = reinterpret_cast<C*>(c->hpart);
    tev_begin(c, 0);
    launch_k(c, gemv_cols<T, NT, true, true, true>, dim3(c->cols_strips, c->dual_S), NT, 0, c->stream, 
        A, c->lda, pfull, qloc, c->nloc, c->n, np, hp, gate);
    c->launches++;
    CK(c, cudaGetLastError());
    launch_k(c, gemv_h_stage2<T, NT, EpiA>, c->nstage2_grid, NT, 0, c->stream, np, c->cols_strips, c->nloc, 0, c->nloc, ea,
                                                                      make_red(c), c->st, gate);
    c->launches++;
    tev_end(c);
    CK(c, cudaGetLastError());
    TRY(post<EpiA>(c, gate));
    if (c->world == 1) {
      launch_k(c, gemv_h_stage2<T, NT, EpiH>, c->stage2_grid, NT, 0, c->stream, hp, c->dual_S, c->n, 0, c->n, eh,
                                                                       make_red(c), c->st, gate);
      c->launches++;
      CK(c, cudaGetLastError());
      return CCG_OK;
    }
    Store<T> stv{reinterpret_cast<C*>(c->wfull)};
    launch_k(c, gemv_h_stage2<T, NT, Store<T>>, c->stage2_grid, NT, 0, c->stream, hp, c->dual_S, c->n, 0, c->n, stv,
                                                                         make_red(c), c->st, gate);
    c->launches++;
    CK(c, cudaGetLastError());
    C* wl = L(c, NLOCAL - 1);
    NK(c, c->comm->reduce_scatter(c->wfull, wl, (size_t)c->nloc * 2, ndt(), c->stream));
    EpiPass<C, EpiH> ep{eh, wl};
    return pass(c, ep, gate);
  }

  // ==================== method schedules ====================
  // local vector slots (NLOCAL-1 is reserved for the multi-GPU Aᴴ result)
  enum { X = 0 };

  static int init_residual(ccg_ctx* c, bool has_x0, C* d0, C* d1, C* d2, C* d3) {
    const int* g = c->zero_gate;
    C* y = L(c, 1);  // y is staged in loc[1] by solve()
    InitR<T> ir{y, d0, d1, d2, d3};
    if (has_x0) {
      // x0 already copied into loc[X]; gather it into full[2]
      Copy<T> cp{L(c, X), Fs(c, 2)};
      TRY(pass(c, cp, g));
      TRY(allgather(c, 2));
      return matvec_a(c, F(c, 2), ir, g);
    }
    return pass(c, ir, g);
  }

  // ---- BiCGSTAB: loc: 0 x, 1 y, 2 r, 3 rt, 4 v, 5 t ; full: 0 p, 1 s
  static int bicgstab_setup(ccg_ctx* c, bool x0) { return init_residual(c, x0, L(c, 2), L(c, 3), nullptr, nullptr); }
  static int bicgstab_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    const int* g2 = &c->st->gate2;
    TRY(pass(c, BsP<T>{L(c, 2), Fs(c, 0), L(c, 4)}, g));
    TRY(allgather(c, 0));
    TRY(matvec_a(c, F(c, 0), BsV<T>{L(c, 4), L(c, 3)}, g));
    TRY(pass(c, BsS<T>{L(c, 2), L(c, 4), Fs(c, 1)}, g));
    TRY(allgather(c, 1));
    TRY(matvec_a(c, F(c, 1), BsT<T>{L(c, 5), Fs(c, 1)}, g2));
    return pass(c, BsX<T>{L(c, X), L(c, 2), Fs(c, 0), Fs(c, 1), L(c, 5), L(c, 3)}, g);
  }

  // ---- CGNE: loc: 0 x, 1 y, 2 r ; full: 0 p
  static int cgne_setup(ccg_ctx* c, bool x0) {
    TRY(init_residual(c, x0, L(c, 2), nullptr, nullptr, nullptr));
    return matvec_h(c, L(c, 2), true, CgP0<T>{Fs(c, 0)}, &c->st->done);
  }
  static int cgne_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    TRY(allgather(c, 0));
    TRY(matvec_a(c, F(c, 0), CgQ<T>{L(c, 2), L(c, X), Fs(c, 0)}, g));
    return matvec_h(c, L(c, 2), true, CgP<T>{Fs(c, 0)}, g);
  }

  // ---- QMR: loc: 0 x, 1 y, 2 r, 3 vt, 4 wt, 5 v, 6 w, 7 q, 8 pt, 9 d, 10 s ; full: 0 p
  static int qmr_setup(ccg_ctx* c, bool x0) {
    TRY(init_residual(c, x0, L(c, 2), L(c, 3), L(c, 4), nullptr));
    return pass(c, QmV<T>{L(c, 3), L(c, 4), L(c, 5), L(c, 6)}, &c->st->done);
  }
  static int qmr_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    TRY(pass(c, QmP<T>{L(c, 5), L(c, 6), Fs(c, 0), L(c, 7)}, g));
    TRY(allgather(c, 0));
    if (c->opk == OPK_DENSE && c->cols_ok && c->qmr_dual && !c->rep && !c->jac_active) {
      TRY(matvec_dual(c, F(c, 0), L(c, 7), QmPt<T>{L(c, 8), L(c, 7)},
                      QmVW<T>{L(c, 3), L(c, 4), L(c, 8), L(c, 5), L(c, 6)}, g));
    } else {
      TRY(matvec_a(c, F(c, 0), QmPt<T>{L(c, 8), L(c, 7)}, g));
      TRY(matvec_h(c, L(c, 7), true, QmVW<T>{L(c, 3), L(c, 4), L(c, 8), L(c, 5), L(c, 6)}, g));
    }
    return pass(c, QmDV<T>{L(c, 9), L(c, 10), L(c, X), L(c, 2), Fs(c, 0), L(c, 8), L(c, 3), L(c, 4), L(c, 5),
                           L(c, 6)},
                g);
  }

  // ---- BiCOR: loc: 0 x, 1 y, 2 rs, 3 rh, 4 p, 5 ps, 6 q, 7 qs ; full: 0 r
  static int bicor_setup(ccg_ctx* c, bool x0) { return init_residual(c, x0, Fs(c, 0), L(c, 2), nullptr, nullptr); }
  static int bicor_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    TRY(allgather(c, 0));
    TRY(matvec_a(c, F(c, 0), RhoEpi<T>{L(c, 3), L(c, 2)}, g));
    TRY(pass(c, BcP<T>{Fs(c, 0), L(c, 2), L(c, 3), L(c, 4), L(c, 5), L(c, 6)}, g));
    TRY(matvec_h(c, L(c, 5), true, BcQs<T>{L(c, 7), L(c, 6)}, g));
    return pass(c, BcX<T>{L(c, X), Fs(c, 0), L(c, 2), L(c, 4), L(c, 6), L(c, 7)}, g);
  }

  // ---- CORS: loc: 0 x, 1 y, 2 r0s, 3 rh, 4 e, 5 eh, 6 h, 7 hh, 8 q ; full: 0 r, 1 qh
  static int cors_setup(ccg_ctx* c, bool x0) { return init_residual(c, x0, Fs(c, 0), L(c, 2), nullptr, nullptr); }
  static int cors_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    TRY(allgather(c, 0));
    TRY(matvec_a(c, F(c, 0), RhoEpi<T>{L(c, 3), L(c, 2)}, g));
    TRY(pass(c, CoP<T>{Fs(c, 0), L(c, 3), L(c, 6), L(c, 7), L(c, 4), L(c, 5), Fs(c, 1)}, g));
    TRY(allgather(c, 1));
    TRY(matvec_a(c, F(c, 1), CoQ<T>{L(c, 8), L(c, 2)}, g));
    return pass(c, CoH<T>{L(c, 4), L(c, 5), Fs(c, 1), L(c, 8), L(c, 6), L(c, 7), L(c, X), Fs(c, 0)}, g);
  }

  // ==================== whole solve loop in one cluster (cluster.cuh) ====================
  template <class M>
  static int launch_cluster(ccg_ctx* c, const M& m) {
    auto kern = cluster_solve<T, M>;
    C* y = L(c, 1);
    ClCommon<T> cm{InitR<T>{y, nullptr, nullptr, nullptr, nullptr}, Copy<T>{L(c, X), Fs(c, 2)},
                   Copy<T>{L(c, X), Fs(c, 2)}, TrueRes<T>{y}, F(c, 2), c->cl_has_x0};
    switch (c->cl_method) {   // r₀ copies, as init_residual() of each method
      case M_BICGSTAB: case M_BICG: case M_CGS: cm.ir.d0 = L(c, 2); cm.ir.d1 = L(c, 3); break;
      case M_CGNE: case M_CGNR: cm.ir.d0 = L(c, 2); break;
      case M_QMR: cm.ir.d0 = L(c, 2); cm.ir.d1 = L(c, 3); cm.ir.d2 = L(c, 4); break;
      case M_BICOR: case M_CORS: cm.ir.d0 = Fs(c, 0); cm.ir.d1 = L(c, 2); break;
      case M_TFQMR: case M_PBICGSTAB: cm.ir.d0 = L(c, 2); cm.ir.d1 = L(c, 3); cm.ir.d2 = Fs(c, 0); break;
      default: cm.ir.d0 = Fs(c, 0); break;   // COCR
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    cfg.blockDim = dim3(CL_NT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = c->stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (c->cluster_size == 0) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      c->cluster_size = 8;
      for (int cs : {16, 8, 4}) {
        cfg.gridDim = dim3(cs);
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) == cudaSuccess && ncl >= 1) {
          c->cluster_size = cs;
          break;
        }
        cudaGetLastError();
      }
      const char* cs = getenv("CCG_CLUSTER_SIZE");
      if (cs) c->cluster_size = std::max(1, std::min(CL_MAX, atoi(cs)));
    } else {
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    cfg.gridDim = dim3(c->cluster_size);
    at[0].val.clusterDim.x = c->cluster_size;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    CK(c, cudaLaunchKernelEx(&cfg, kern, m, cm, c->st, reinterpret_cast<const C*>(c->A), c->lda, c->n));
    c->launches++;
    return CCG_OK;
  }

  static int cluster_run(ccg_ctx* c, int m) {
    switch (m) {
      case M_BICGSTAB:
        return launch_cluster(c, ClBicgstab<T>{BsP<T>{L(c, 2), Fs(c, 0), L(c, 4)}, BsV<T>{L(c, 4), L(c, 3)},
                                               BsS<T>{L(c, 2), L(c, 4), Fs(c, 1)}, BsT<T>{L(c, 5), Fs(c, 1)},
                                               BsX<T>{L(c, X), L(c, 2), Fs(c, 0), Fs(c, 1), L(c, 5), L(c, 3)},
                                               F(c, 0), F(c, 1)});
      case M_CGNE:
        return launch_cluster(c, ClCgne<T>{CgQ<T>{L(c, 2), L(c, X), Fs(c, 0)}, CgP<T>{Fs(c, 0)}, CgP0<T>{Fs(c, 0)},
                                           F(c, 0), L(c, 2)});
      case M_QMR:
        return launch_cluster(
            c, ClQmr<T>{QmP<T>{L(c, 5), L(c, 6), Fs(c, 0), L(c, 7)}, QmPt<T>{L(c, 8), L(c, 7)},
                        QmVW<T>{L(c, 3), L(c, 4), L(c, 8), L(c, 5), L(c, 6)},
                        QmDV<T>{L(c, 9), L(c, 10), L(c, X), L(c, 2), Fs(c, 0), L(c, 8), L(c, 3), L(c, 4), L(c, 5),
                                L(c, 6)},
                        QmV<T>{L(c, 3), L(c, 4), L(c, 5), L(c, 6)}, F(c, 0), L(c, 7)});
      case M_BICOR:
        return launch_cluster(c, ClBicor<T>{RhoEpi<T>{L(c, 3), L(c, 2)},
                                            BcP<T>{Fs(c, 0), L(c, 2), L(c, 3), L(c, 4), L(c, 5), L(c, 6)},
                                            BcQs<T>{L(c, 7), L(c, 6)},
                                            BcX<T>{L(c, X), Fs(c, 0), L(c, 2), L(c, 4), L(c, 6), L(c, 7)}, F(c, 0),
                                            L(c, 5)});
      case M_CORS:
        return launch_cluster(
            c, ClCors<T>{RhoEpi<T>{L(c, 3), L(c, 2)}, CoP<T>{Fs(c, 0), L(c, 3), L(c, 6), L(c, 7), L(c, 4), L(c, 5), Fs(c, 1)},
                         CoQ<T>{L(c, 8), L(c, 2)},
                         CoH<T>{L(c, 4), L(c, 5), Fs(c, 1), L(c, 8), L(c, 6), L(c, 7), L(c, X), Fs(c, 0)}, F(c, 0),
                         F(c, 1)});
      case M_BICG:
        return launch_cluster(c, ClBicg<T>{BgP<T>{L(c, 2), L(c, 3), Fs(c, 0), L(c, 4)}, BgQ<T>{L(c, 5), L(c, 4)},
                                           Store<T>{L(c, 6)},
                                           BgX<T>{L(c, X), L(c, 2), L(c, 3), Fs(c, 0), L(c, 5), L(c, 6)}, F(c, 0),
                                           L(c, 4)});
      case M_CGS:
        return launch_cluster(c, ClCgs<T>{CsP<T>{L(c, 2), L(c, 5), Fs(c, 0), L(c, 4)}, CsV<T>{L(c, 6), L(c, 3)},
                                          CsQ<T>{L(c, 4), L(c, 6), L(c, 5), Fs(c, 1), L(c, X)},
                                          CsR<T>{L(c, 2), L(c, 3)}, F(c, 0), F(c, 1)});
      case M_COCR:
        return launch_cluster(c, ClCocr<T>{CrP<T>{Fs(c, 0), L(c, 2), L(c, 3), L(c, 4)},
                                           CrX<T>{L(c, X), Fs(c, 0), L(c, 3), L(c, 4)}, CrAr<T>{L(c, 2), Fs(c, 0)},
                                           CrAr0<T>{L(c, 2), Fs(c, 0)}, F(c, 0)});
      case M_TFQMR:
        return launch_cluster(c, ClTfqmr<T>{TfE<T>{Fs(c, 0), L(c, 4), L(c, 6), Fs(c, 1), L(c, 3), L(c, 5)},
                                            TfO<T>{L(c, 7), L(c, X), L(c, 3), L(c, 5), Fs(c, 1), L(c, 2)},
                                            TfU<T>{L(c, X), L(c, 5), L(c, 3), Fs(c, 1), Fs(c, 0)},
                                            TfV<T>{L(c, 6), L(c, 7), L(c, 4), L(c, 2)},
                                            TfV0<T>{L(c, 4), L(c, 6), L(c, 2)}, F(c, 0), F(c, 1)});
      case M_PBICGSTAB:
        return launch_cluster(
            c, ClPbicgstab<T>{PbW0<T>{Fs(c, 1), L(c, 3)}, PbStore<T>{L(c, 9)},
                              PbP1<T>{L(c, 2), Fs(c, 1), L(c, 9), L(c, 8), L(c, 4), L(c, 5), Fs(c, 0), L(c, 6), L(c, 7)},
                              PbStore<T>{L(c, 8)},
                              PbP2<T>{L(c, X), L(c, 2), Fs(c, 1), L(c, 4), L(c, 6), L(c, 7), L(c, 9), L(c, 8), L(c, 5),
                                      Fs(c, 0), L(c, 3)},
                              PbT<T>{L(c, 9)}, F(c, 0), F(c, 1)});
      default:
        return launch_cluster(c, ClCgnr<T>{CnW<T>{L(c, 3)}, CnX<T>{L(c, X), L(c, 2), Fs(c, 0), L(c, 3)},
                                           CnZ<T>{L(c, 4)}, CnP<T>{L(c, 4), Fs(c, 0)}, CnZ0<T>{Fs(c, 0)}, F(c, 0),
                                           L(c, 2)});
    }
  }

  // ==================== SURVEY §8(f) NEXT-3 ====================
  // A·p and Aᴴ·p̃ of one BiCG iteration are independent: dual GEMV when dense
  template <class EpiA, class EpiH>
  static int matvec_pair(ccg_ctx* c, int pfull_idx, const C* qloc, EpiA ea, EpiH eh, const int* gate) {
    if (c->opk == OPK_DENSE && c->cols_ok && c->qmr_dual && !c->rep && !c->jac_active)
      return matvec_dual(c, F(c, pfull_idx), qloc, ea, eh, gate);
    TRY(matvec_a(c, F(c, pfull_idx), ea, gate));
    return matvec_h(c, qloc, true, eh, gate);
  }

  // ---- BiCG: loc: 0 x, 1 y, 2 r, 3 rt, 4 pt, 5 q, 6 qt ; full: 0 p
  static int bicg_setup(ccg_ctx* c, bool x0) { return init_residual(c, x0, L(c, 2), L(c, 3), nullptr, nullptr); }
  static int bicg_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    TRY(pass(c, BgP<T>{L(c, 2), L(c, 3), Fs(c, 0), L(c, 4)}, g));
    TRY(allgather(c, 0));
    TRY(matvec_pair(c, 0, L(c, 4), BgQ<T>{L(c, 5), L(c, 4)}, Store<T>{L(c, 6)}, g));
    return pass(c, BgX<T>{L(c, X), L(c, 2), L(c, 3), Fs(c, 0), L(c, 5), L(c, 6)}, g);
  }

  // ---- CGS: loc: 0 x, 1 y, 2 r, 3 rt, 4 u, 5 q, 6 v ; full: 0 p, 1 u+q
  static int cgs_setup(ccg_ctx* c, bool x0) { return init_residual(c, x0, L(c, 2), L(c, 3), nullptr, nullptr); }
  static int cgs_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    TRY(pass(c, CsP<T>{L(c, 2), L(c, 5), Fs(c, 0), L(c, 4)}, g));
    TRY(allgather(c, 0));
    TRY(matvec_a(c, F(c, 0), CsV<T>{L(c, 6), L(c, 3)}, g));
    TRY(pass(c, CsQ<T>{L(c, 4), L(c, 6), L(c, 5), Fs(c, 1), L(c, X)}, g));
    TRY(allgather(c, 1));
    return matvec_a(c, F(c, 1), CsR<T>{L(c, 2), L(c, 3)}, g);
  }

  // ---- COCR: loc: 0 x, 1 y, 2 Ar, 3 p, 4 Ap ; full: 0 r
  static int cocr_setup(ccg_ctx* c, bool x0) {
    TRY(init_residual(c, x0, Fs(c, 0), nullptr, nullptr, nullptr));
    TRY(allgather(c, 0));
    return matvec_a(c, F(c, 0), CrAr0<T>{L(c, 2), Fs(c, 0)}, &c->st->done);
  }
  static int cocr_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    TRY(pass(c, CrP<T>{Fs(c, 0), L(c, 2), L(c, 3), L(c, 4)}, g));
    TRY(pass(c, CrX<T>{L(c, X), Fs(c, 0), L(c, 3), L(c, 4)}, g));
    TRY(allgather(c, 0));
    return matvec_a(c, F(c, 0), CrAr<T>{L(c, 2), Fs(c, 0)}, g);
  }

  // ---- CGNR: loc: 0 x, 1 y, 2 r, 3 w, 4 z ; full: 0 p
  static int cgnr_setup(ccg_ctx* c, bool x0) {
    TRY(init_residual(c, x0, L(c, 2), nullptr, nullptr, nullptr));
    return matvec_h(c, L(c, 2), true, CnZ0<T>{Fs(c, 0)}, &c->st->done);
  }
  static int cgnr_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    TRY(allgather(c, 0));
    TRY(matvec_a(c, F(c, 0), CnW<T>{L(c, 3)}, g));
    TRY(pass(c, CnX<T>{L(c, X), L(c, 2), Fs(c, 0), L(c, 3)}, g));
    TRY(matvec_h(c, L(c, 2), true, CnZ<T>{L(c, 4)}, g));
    return pass(c, CnP<T>{L(c, 4), Fs(c, 0)}, g);
  }

  // ---- TFQMR: loc: 0 x, 1 y, 2 r0*, 3 w, 4 v, 5 d, 6 A·u (even), 7 A·u2 ; full: 0 u, 1 u2
  static int tfqmr_setup(ccg_ctx* c, bool x0) {
    TRY(init_residual(c, x0, L(c, 2), L(c, 3), Fs(c, 0), nullptr));
    TRY(allgather(c, 0));
    return matvec_a(c, F(c, 0), TfV0<T>{L(c, 4), L(c, 6), L(c, 2)}, &c->st->done);
  }
  static int tfqmr_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    const int* g2 = &c->st->gate2;
    TRY(pass(c, TfE<T>{Fs(c, 0), L(c, 4), L(c, 6), Fs(c, 1), L(c, 3), L(c, 5)}, g));
    TRY(allgather(c, 1));
    TRY(matvec_a(c, F(c, 1), TfO<T>{L(c, 7), L(c, X), L(c, 3), L(c, 5), Fs(c, 1), L(c, 2)}, g2));
    TRY(pass(c, TfU<T>{L(c, X), L(c, 5), L(c, 3), Fs(c, 1), Fs(c, 0)}, g));
    TRY(allgather(c, 0));
    return matvec_a(c, F(c, 0), TfV<T>{L(c, 6), L(c, 7), L(c, 4), L(c, 2)}, g);
  }

  // ---- GMRES(m): loc: 0 x, 1 y, 2 w ; basis V (gm_V) ; full: 0 v_j, 2 x (restart)
  static C* Vb(ccg_ctx* c) { return reinterpret_cast<C*>(c->gm_V); }
  template <int MODE>
  static int gm_pass_launch(ccg_ctx* c, C* w, const double2* coef, double2* dst, const int* gate) {
    const bool fuse = c->world == 1 || c->rep;
    auto kern = c->gm_fast ? gm_pass<T, MODE, true> : gm_pass<T, MODE, false>;
    launch_k(c, kern, c->gm_grid, GM_NT, 0, c->stream, Vb(c), c->nloc, w, coef, fuse ? dst : c->gm_rank, c->nloc,
             c->gm_dev, c->gm_part, c->gm_ticket, fuse ? 1 : 0, gate);
    c->launches++;
    CK(c, cudaGetLastError());
    if (!fuse) {
      NK(c, c->comm->allgather(c->gm_rank, c->gm_all, (size_t)(GM_MAX + 1) * 2, CT_F64, c->stream));
      launch_k(c, gm_ranksum, 1, 128, 0, c->stream, c->gm_all, c->world, MODE == 2 ? 1 : GM_MAX + 1, GM_MAX + 1, dst, gate);
      c->launches++;
    }
    return CCG_OK;
  }
  static int gmres_setup(ccg_ctx* c, bool x0) {
    TRY(init_residual(c, x0, Vb(c), nullptr, nullptr, nullptr));
    launch_k(c, gm_normalize<T>, c->gm_vgrid, NT, 0, c->stream, Vb(c), c->nloc, Vb(c), Fs(c, 0), c->nloc, c->gm_dev, 1,
                                                         &c->st->done);
    c->launches++;
    CK(c, cudaGetLastError());
    return CCG_OK;
  }
  static int gmres_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    GmDev* gm = c->gm_dev;
    C* w = L(c, 2);
    TRY(allgather(c, 0));
    TRY(matvec_a(c, F(c, 0), Store<T>{w}, g));
    TRY(gm_pass_launch<0>(c, w, nullptr, gm->hcol, g));
    TRY(gm_pass_launch<1>(c, w, gm->hcol, gm->h2, g));
    TRY(gm_pass_launch<2>(c, w, gm->h2, &gm->ww2, g));
    launch_k(c, gm_step, 1, 1, 0, c->stream, c->st, gm, g);
    launch_k(c, gm_normalize<T>, c->gm_vgrid, NT, 0, c->stream, Vb(c), c->nloc, w, Fs(c, 0), c->nloc, gm, 0, &gm->endflag);
    launch_k(c, gm_trisolve, 1, 1, 0, c->stream, c->st, gm, &gm->noend);
    launch_k(c, gm_xupdate<T>, c->gm_vgrid, NT, 0, c->stream, L(c, X), Vb(c), c->nloc, c->nloc, gm, &gm->noxupd);
    c->launches += 4;
    CK(c, cudaGetLastError());
    TRY(pass(c, Copy<T>{L(c, X), Fs(c, 2)}, &gm->norestart));
    TRY(allgather(c, 2));
    TRY(matvec_a(c, F(c, 2), GmR<T>{L(c, 1), Vb(c)}, &gm->norestart));
    launch_k(c, gm_normalize<T>, c->gm_vgrid, NT, 0, c->stream, Vb(c), c->nloc, Vb(c), Fs(c, 0), c->nloc, gm, 1,
                                                         &gm->norestart);
    launch_k(c, gm_reset, 1, 1, 0, c->stream, gm);
    c->launches += 2;
    CK(c, cudaGetLastError());
    return CCG_OK;
  }

  // ---- BiCGstab(ℓ): loc: 0 x, 1 y, 3 r̃ ; bl_buf: r̂₀..r̂_ℓ then û₀..û_ℓ (full length each)
  static C* BLR(ccg_ctx* c, int a) { return reinterpret_cast<C*>(c->bl_buf) + (size_t)a * c->n; }
  static C* BLU(ccg_ctx* c, int a) { return BLR(c, c->bl_l + 1 + a); }
  static C* BRs(ccg_ctx* c, int a) { return BLR(c, a) + c->row0; }
  static C* BUs(ccg_ctx* c, int a) { return BLU(c, a) + c->row0; }
  static int allgather_buf(ccg_ctx* c, C* buf) {
    if (c->world == 1 || c->rep) return CCG_OK;
    if (c->opk == OPK_CSR || c->opk == OPK_STENCIL) return halo_exchange(c, buf);
    NK(c, c->comm->allgather_inplace(buf, (size_t)c->nloc * 2, ndt(), c->stream));
    return CCG_OK;
  }
  static int bicgstabl_setup(ccg_ctx* c, bool x0) {
    TRY(init_residual(c, x0, BRs(c, 0), L(c, 3), nullptr, nullptr));
    CK(c, cudaMemsetAsync(BUs(c, 0), 0, (size_t)c->nloc * sizeof(C), c->stream));
    return CCG_OK;
  }
  template <int LL>
  static int bicgstabl_mr(ccg_ctx* c, const int* g) {
    BlGram<T, LL> G{};
    BlM<T, LL> M{};
    for (int a = 0; a <= LL; ++a) {
      G.r[a] = BRs(c, a);
      M.r[a] = BRs(c, a);
      M.u[a] = BUs(c, a);
    }
    M.x = L(c, X);
    M.rt = L(c, 3);
    TRY(pass(c, G, g));
    return pass(c, M, g);
  }
  static int bicgstabl_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    const int ell = c->bl_l;
    for (int j = 0; j < ell; ++j) {
      BlP<T> P{};
      for (int a = 0; a <= j; ++a) { P.u[a] = BUs(c, a); P.r[a] = BRs(c, a); }
      P.J = j;
      TRY(pass(c, P, g));
      TRY(allgather_buf(c, BLU(c, j)));
      TRY(matvec_a(c, BLU(c, j), BlU<T>{BUs(c, j + 1), L(c, 3)}, g));
      BlX<T> Xp{};
      for (int a = 0; a <= j; ++a) Xp.r[a] = BRs(c, a);
      for (int a = 0; a <= j + 1; ++a) Xp.u[a] = BUs(c, a);
      Xp.x = L(c, X);
      Xp.J = j;
      TRY(pass(c, Xp, g));
      TRY(allgather_buf(c, BLR(c, j)));
      if (j < ell - 1)
        TRY(matvec_a(c, BLR(c, j), BlR<T>{BRs(c, j + 1), L(c, 3)}, g));
      else
        TRY(matvec_a(c, BLR(c, j), BlRL<T>{BRs(c, j + 1)}, g));
    }
    switch (ell) {
      case 1: return bicgstabl_mr<1>(c, g);
      case 2: return bicgstabl_mr<2>(c, g);
      case 3: return bicgstabl_mr<3>(c, g);
      default: return bicgstabl_mr<4>(c, g);
    }
  }

  // ---- p-BiCGSTAB: loc: 0 x, 1 y, 2 r, 3 r̃, 4 p, 5 s, 6 q, 7 y, 8 v, 9 t ; full: 0 z (r₀ at setup), 1 w
  static int pbicgstab_setup(ccg_ctx* c, bool x0) {
    const int* g = &c->st->done;
    TRY(init_residual(c, x0, L(c, 2), L(c, 3), Fs(c, 0), nullptr));
    TRY(allgather(c, 0));
    TRY(matvec_a(c, F(c, 0), PbW0<T>{Fs(c, 1), L(c, 3)}, g));
    TRY(allgather(c, 1));
    return matvec_a(c, F(c, 1), PbStore<T>{L(c, 9)}, g);
  }
  static int pbicgstab_iter(ccg_ctx* c) {
    const int* g = &c->st->done;
    const int* g2 = &c->st->gate2;
    TRY(pass(c, PbP1<T>{L(c, 2), Fs(c, 1), L(c, 9), L(c, 8), L(c, 4), L(c, 5), Fs(c, 0), L(c, 6), L(c, 7)}, g));
    TRY(allgather(c, 0));
    TRY(matvec_a(c, F(c, 0), PbStore<T>{L(c, 8)}, g2));
    TRY(pass(c, PbP2<T>{L(c, X), L(c, 2), Fs(c, 1), L(c, 4), L(c, 6), L(c, 7), L(c, 9), L(c, 8), L(c, 5), Fs(c, 0),
                        L(c, 3)},
             g));
    TRY(allgather(c, 1));
    return matvec_a(c, F(c, 1), PbT<T>{L(c, 9)}, g);
  }

  static int setup(ccg_ctx* c, int m, bool x0) {
    switch (m) {
      case M_BICGSTAB: return bicgstab_setup(c, x0);
      case M_CGNE: return cgne_setup(c, x0);
      case M_QMR: return qmr_setup(c, x0);
      case M_BICOR: return bicor_setup(c, x0);
      case M_CORS: return cors_setup(c, x0);
      case M_BICG: return bicg_setup(c, x0);
      case M_CGS: return cgs_setup(c, x0);
      case M_COCR: return cocr_setup(c, x0);
      case M_TFQMR: return tfqmr_setup(c, x0);
      case M_GMRES: return gmres_setup(c, x0);
      case M_BICGSTABL: return bicgstabl_setup(c, x0);
      case M_PBICGSTAB: return pbicgstab_setup(c, x0);
      default: return cgnr_setup(c, x0);
    }
  }
  static int iter(ccg_ctx* c, int m) {
    switch (m) {
      case M_BICGSTAB: return bicgstab_iter(c);
      case M_CGNE: return cgne_iter(c);
      case M_QMR: return qmr_iter(c);
      case M_BICOR: return bicor_iter(c);
      case M_CORS: return cors_iter(c);
      case M_BICG: return bicg_iter(c);
      case M_CGS: return cgs_iter(c);
      case M_COCR: return cocr_iter(c);
      case M_TFQMR: return tfqmr_iter(c);
      case M_GMRES: return gmres_iter(c);
      case M_BICGSTABL: return bicgstabl_iter(c);
      case M_PBICGSTAB: return pbicgstab_iter(c);
      default: return cgnr_iter(c);
    }
  }

  // true residual ‖y − A x‖²
  static int true_residual(ccg_ctx* c) {
    const int* g = c->zero_gate;
    TRY(pass(c, Copy<T>{L(c, X), Fs(c, 2)}, g));
    TRY(allgather(c, 2));
    return matvec_a(c, F(c, 2), TrueRes<T>{L(c, 1)}, g);
  }

  // right Jacobi around a solve: u₀ = D·x₀ before, x = D⁻¹·u after
  static int jac_in(ccg_ctx* c) {
    return pass_count(c, JacScale<T>{L(c, X), reinterpret_cast<const C*>(c->jac_d) + c->row0, L(c, X)}, c->nloc,
                      c->zero_gate);
  }
  static int jac_out(ccg_ctx* c) {
    return pass_count(c, JacScale<T>{L(c, X), reinterpret_cast<const C*>(c->jac_dinv) + c->row0, L(c, X)}, c->nloc,
                      c->zero_gate);
  }

  // ccg_apply
  static int apply(ccg_ctx* c, int op, const C* xin, C* yout) {
    const int* g = c->zero_gate;
    if (op == CCG_OP_A || (op == CCG_OP_AT && (c->opk == OPK_CSR || c->opk == OPK_STENCIL))) {
      CK(c, cudaMemcpyAsync(Fs(c, 2), xin, c->nloc * sizeof(C), cudaMemcpyDeviceToDevice, c->stream));
      TRY(allgather(c, 2));
      return matvec_a(c, F(c, 2), Store<T>{yout}, g);
    }
    CK(c, cudaMemcpyAsync(L(c, 2), xin, c->nloc * sizeof(C), cudaMemcpyDeviceToDevice, c->stream));
    return matvec_h(c, L(c, 2), op == CCG_OP_AH, Store<T>{yout}, g);
  }
};

// ===========================================================================
// launch-parameter selection
// ===========================================================================
// Row splits S for a (strips × S) grid of column-owner CTAs: the smallest S ≥
// ceil(slots/strips) whose grid fills its last wave to ≥ 90 % (wave
// quantisation), at most 128 and at most max_rows_split (≥ 16 rows per split).
static int64_t pick_splits(int64_t strips, int64_t slots, int64_t max_split) {
  max_split = std::max<int64_t>(1, std::min<int64_t>(max_split, 128));
  int64_t S0 = std::max<int64_t>(1, (slots + strips - 1) / strips);
  if (S0 >= max_split) return max_split;
  for (int64_t S = S0; S <= std::min<int64_t>(max_split, 4 * S0); ++S) {
    const int64_t ctas = strips * S;
    const int64_t waves = (ctas + slots - 1) / slots;
    if (ctas >= (int64_t)(0.9 * waves * slots)) return S;
  }
  return S0;
}
template <typename T>
static int choose_launch(ccg_ctx* c) {
  using E = Engine<T>;
  using C = typename CT<T>::c;
  const int NT = E::NT;
  int occ = 0;
  if (c->vec_ok)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemv_n_kernel<T, E::R, E::NT, true, Store<T>>, NT, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemv_n_kernel<T, E::R, E::NT, false, Store<T>>, NT, 0);
  if (occ < 1) occ = 1;
  const int64_t groups = (c->mnloc + E::R - 1) / E::R;
  c->gemv_grid = (int)std::max<int64_t>(1, std::min<int64_t>(groups, (int64_t)c->sm_count * occ));
  c->bulk_ok = c->opk == OPK_DENSE && getenv("CCG_NO_BULK") == nullptr &&
               ((c->n * (int64_t)sizeof(C)) % BULK_TILE == 0) && ((c->lda * (int64_t)sizeof(C)) % 16 == 0) &&
               (((uintptr_t)c->A) % 16 == 0);
  c->bulk_grid = (int)std::max<int64_t>(1, std::min<int64_t>((c->mnloc + E::BR - 1) / E::BR, c->sm_count));
  {
    const char* gm = getenv("CCG_GEMV");
    c->gemv_mode = (gm && !strcmp(gm, "bulk"))    ? GEMV_BULK
                   : (gm && !strcmp(gm, "rows"))  ? GEMV_ROWS
                   : (gm && !strcmp(gm, "cols"))  ? GEMV_COLS
                   // default: the split kernel (config 3: 7.19 vs 6.99 TB/s for the
                   // column-owner layout; config 2 whole solves in an interleaved
                   // A/B: BiCGSTAB 120.5 vs 124.5 µs/it, COCR 63.7 vs 65.7 —
                   // profiles/r01/ab/cfg2_gemv.jsonl)
                   : GEMV_SPLIT;
    const char* qd = getenv("CCG_QMR_DUAL");
    c->qmr_dual = !(qd && !strcmp(qd, "0"));
  }
  // column-owner GEMV (A·x in GEMV_COLS mode; QMR dual product): strips of NT·V
  // columns; A·x alone: whole waves of (strip, split) CTAs; dual: as for Aᴴ
  c->cols_ok = c->opk == OPK_DENSE && c->vec_ok && (c->n % CT<T>::V) == 0;
  if (c->cols_ok) {
    const int64_t nvc = c->n / CT<T>::V;
    c->cols_strips = (int)std::max<int64_t>(1, (nvc + NT - 1) / NT);
    const char* rg = getenv("CCG_COLS_RG");
    c->cols_rg = (rg && atoi(rg) == 4) ? 4 : 1;
    int occc = 0;
    if (c->cols_rg == 4)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occc, gemv_cols<T, E::NT, true, false, false, 4>, NT, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occc, gemv_cols<T, E::NT, true, false, false, 1>, NT, 0);
    if (occc < 1) occc = 1;
    const int64_t slots_c = (int64_t)c->sm_count * occc;
    const char* wv = getenv("CCG_COLS_WAVES");
    const int64_t waves = wv ? std::max(1, atoi(wv)) : 2;
    int64_t Sn = std::max<int64_t>(1, (waves * slots_c) / c->cols_strips);
    c->cols_S = (int)std::min<int64_t>(Sn, std::max<int64_t>(1, c->mnloc / 8));
    int occd = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occd, gemv_cols<T, E::NT, true, true, true>, NT, 0);
    if (occd < 1) occd = 1;
    c->dual_S = (int)pick_splits(c->cols_strips, (int64_t)c->sm_count * occd, c->mnloc / 16);
    c->nstage2_grid =
        (int)std::max<int64_t>(1, std::min<int64_t>((c->mnloc + NT - 1) / NT, (int64_t)c->sm_count * 4));
    size_t need = (size_t)c->cols_strips * c->mnloc * sizeof(C);
    if (need > c->npart_bytes) {
      if (c->npart) cudaFree(c->npart);
      c->npart = nullptr;
      CK(c, cudaMalloc(&c->npart, need));
      c->npart_bytes = need;
    }
  }
  if (c->opk == OPK_DENSE && c->gemv_mode == GEMV_SPLIT) {
    // x strip of 16 KiB in shared memory; whole waves of CTAs (strips × row blocks)
    // (CCG_SPLIT_KB / CCG_SPLIT_UR / CCG_SPLIT_WAVES: tuning knobs for sweeps)
    const char* kb = getenv("CCG_SPLIT_KB");
    const char* ur = getenv("CCG_SPLIT_UR");
    const char* wv = getenv("CCG_SPLIT_WAVES");
    const int64_t strip_bytes = kb ? std::max(1, atoi(kb)) * 1024 : 16384;
    c->split_ur = ur ? atoi(ur) : 8;
    const int max_waves = wv ? std::max(1, atoi(wv)) : 4;
    c->split_W = (int)std::min<int64_t>(c->n, strip_bytes / (int64_t)sizeof(C));
    c->split_strips = (int)((c->n + c->split_W - 1) / c->split_W);
    int occs = 0;
    if (c->vec_ok)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs, gemv_n_split<T, E::NT, E::SUR, true, false, Store<T>>,
                                                    NT, (size_t)c->split_W * sizeof(C));
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs, gemv_n_split<T, E::NT, E::SUR, false, false, Store<T>>,
                                                    NT, (size_t)c->split_W * sizeof(C));
    if (occs < 1) occs = 1;
    const int64_t slots = (int64_t)c->sm_count * occs;
    // waves k: row blocks of >= 64 rows (x-strip reuse), CTAs = k·slots
    int64_t nrb = 1;
    for (int k = max_waves; k >= 1; --k) {
      nrb = std::max<int64_t>(1, (k * slots) / c->split_strips);
      if (c->mnloc / nrb >= 64 || k == 1) break;
    }
    nrb = std::min<int64_t>(nrb, std::max<int64_t>(1, c->mnloc / 8));
    c->split_nrb = (int)nrb;
    c->nstage2_grid =
        (int)std::max<int64_t>(1, std::min<int64_t>((c->mnloc + NT - 1) / NT, (int64_t)c->sm_count * 4));
    size_t need = c->split_strips > 1 ? (size_t)c->split_strips * c->mnloc * sizeof(C) : 0;
    if (need > c->npart_bytes) {
      if (c->npart) cudaFree(c->npart);
      c->npart = nullptr;
      CK(c, cudaMalloc(&c->npart, need));
      c->npart_bytes = need;
    }
  }
  // Aᴴ stage 1: strips of NT*V columns, S row splits, ~ whole waves
  const int V = c->vec_ok ? CT<T>::V : 1;
  const int64_t nv = c->n / V;
  c->ah_strips = (int)std::max<int64_t>(1, (nv + NT - 1) / NT);
  int occ1 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, gemv_h_stage1<T, true, E::NT, E::UR, true>, NT, 0);
  if (occ1 < 1) occ1 = 1;
  const int64_t slots = (int64_t)c->sm_count * occ1;
  int64_t S = slots / c->ah_strips;
  S = std::max<int64_t>(1, std::min<int64_t>(S, 128));
  S = std::min<int64_t>(S, std::max<int64_t>(1, c->mnloc / 16));
  c->ah_S = (int)S;
  c->stage2_grid = (int)std::max<int64_t>(1, std::min<int64_t>((c->n + NT - 1) / NT, (int64_t)c->sm_count * 4));
  c->pass_grid = (int)std::max<int64_t>(1, std::min<int64_t>((c->nloc + NT - 1) / NT, (int64_t)c->sm_count * 8));
  c->spmv_grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((c->mnloc + NT / E::LPR - 1) / (NT / E::LPR), (int64_t)c->sm_count * 8));
  if (c->sell_col) {
    // measured (tools/sweep_sell.py, interleaved medians, profiles/r01/
    // sweep_sell.jsonl): one row per step at ≥ 3 CTAs/SM wins for both dtypes
    // (config 5 COCR c128 172.6 → 135.6 µs/it, c64 87.7 → 84.3)
    c->sell_one = 1;
    const char* sm = getenv("CCG_SELL_ONE");
    if (sm) c->sell_one = atoi(sm) != 0;
    const char* sw = getenv("CCG_SELL_WAVES");
    if (sw) c->sell_waves = std::max(1, std::min(64, atoi(sw)));
    int occ4[2] = {0, 0};
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ4[0], spmv_sell_kernel<T, E::NT, false, false, Store<T>>, NT, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ4[1], spmv_sell_kernel<T, E::NT, false, true, Store<T>>, NT, 0);
    const int64_t thr = ((c->mnloc + 31) / 32) * 32;
    for (int m = 0; m < 2; ++m)
      c->sell_grid[m] = (int)std::max<int64_t>(
          1, std::min<int64_t>((thr + NT - 1) / NT, (int64_t)c->sm_count * std::max(1, occ4[m]) * c->sell_waves));
  }
  if (c->csr_blocks) {
    int occ3 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, spmv_stream_kernel<T, E::NT, E::SNNZ, false, Store<T>>,
                                                  NT, 0);
    if (occ3 < 1) occ3 = 1;
    c->spmv_grid = (int)std::max<int64_t>(1, std::min<int64_t>(c->csr_nblocks, (int64_t)c->sm_count * occ3));
  }
  // workspace sized for the chosen grids
  size_t need_hpart = (size_t)std::max(c->ah_S, c->cols_ok ? c->dual_S : 1) * (size_t)c->n * sizeof(C);
  if (c->opk == OPK_DENSE && need_hpart > c->hpart_bytes) {
    if (c->hpart) cudaFree(c->hpart);
    c->hpart = nullptr;
    CK(c, cudaMalloc(&c->hpart, need_hpart));
    c->hpart_bytes = need_hpart;
  }
  int64_t maxgrid = std::max<int64_t>({(int64_t)c->gemv_grid, (int64_t)c->ah_strips * c->ah_S,
                                       (int64_t)c->stage2_grid, (int64_t)c->pass_grid, (int64_t)c->spmv_grid,
                                       (int64_t)c->split_strips * c->split_nrb, (int64_t)c->nstage2_grid,
                                       (int64_t)c->bulk_grid, (int64_t)std::max(c->sell_grid[0], c->sell_grid[1]),
                                       (int64_t)c->cols_strips * std::max(c->cols_S, c->dual_S),
                                       c->opk == OPK_STENCIL ? (int64_t)((c->snx + 31) / 32) * ((c->sny + 7) / 8) *
                                                                   ((c->snzl + c->szc - 1) / c->szc)
                                                             : (int64_t)1,
                                       c->opk == OPK_TOEPLITZ
                                           ? (int64_t)(c->geo.ny * c->geo.nz + c->geo.tx - 1) / c->geo.tx
                                           : (int64_t)1});
  size_t need_part = (size_t)maxgrid * 16;   // up to 16 partial sums per CTA (BiCGstab(ℓ) Gram pass)
  if (need_part > c->part_cap) {
    if (c->part) cudaFree(c->part);
    c->part = nullptr;
    CK(c, cudaMalloc(&c->part, need_part * sizeof(double2)));
    c->part_cap = need_part;
  }
  return CCG_OK;
}

static void free_csr_copies(ccg_ctx* c) {
  if (c->cb_out) cudaFree(c->cb_out);
  c->cb_out = nullptr;
  if (c->fftW) cudaFree(c->fftW);
  if (c->fftK) cudaFree(c->fftK);
  if (c->fftTw) cudaFree(c->fftTw);
  c->fftW = c->fftK = c->fftTw = nullptr;
  if (c->csr_blocks) cudaFree(c->csr_blocks);
  if (c->sell_off) cudaFree(c->sell_off);
  if (c->sell_width) cudaFree(c->sell_width);
  if (c->sell_col) cudaFree(c->sell_col);
  if (c->sell_val) cudaFree(c->sell_val);
  c->csr_blocks = nullptr;
  c->csr_nblocks = 0;
  c->sell_off = nullptr;
  c->sell_width = nullptr;
  c->sell_col = nullptr;
  c->sell_val = nullptr;
}

static void invalidate_graphs(ccg_ctx* c) {
  for (int m = 0; m < M_COUNT; ++m) {
    if (c->gexec[m]) cudaGraphExecDestroy(c->gexec[m]);
    c->gexec[m] = nullptr;
  }
}

// ===========================================================================
// C-ABI
// ===========================================================================
template <typename T>
static int run_iterations(ccg_ctx* c, int m, int maxit) {
  using E = Engine<T>;
  int done = 0;
  auto read_done = [&]() -> int {
    CK(c, cudaMemcpyAsync(&c->st_host->done, &c->st->done, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    done = c->st_host->done;
    return CCG_OK;
  };
  TRY(read_done());
  if (done) return CCG_OK;
  const bool eager_cb = c->opk == OPK_CALLBACK && !(c->cb_caps & CCG_CB_GRAPH_SAFE);
  if (c->timing || eager_cb || (c->comm && !c->comm->graph_safe)) {
    for (int k = 0; k < maxit && !done; ++k) {
      TRY(E::iter(c, m));
      TRY(read_done());
      tev_collect(c);
    }
    return CCG_OK;
  }
  if (!c->gexec[m]) {
    cudaGraph_t graph;
    int64_t l0 = c->launches;
    CK(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int rc = E::iter(c, m);
    cudaError_t e2 = cudaStreamEndCapture(c->stream, &graph);
    if (rc) return rc;
    if (e2 != cudaSuccess) FAIL(c, CCG_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e2));
    c->graph_launches_per_iter[m] = c->launches - l0;
    c->launches = l0;
    CK(c, cudaGraphInstantiate(&c->gexec[m], graph, 0));
    cudaGraphDestroy(graph);
  }
  // Chunks of `chunk` graph launches, each followed by an async copy of the
  // done flag + an event; the host waits for that chunk's flag (~200 µs of
  // work per chunk).  Iterations queued after convergence are gated on the
  // device flag and return at once.  CCG_PIPELINE=1 queues chunk j+1 before
  // waiting for chunk j (no GPU idle on the host round trip, but a whole
  // gated chunk after convergence): measured ±2 % on long solves and up to
  // 12 % slower on short ones, so it is off by default.
  int k = 0, chunk = 1, pending = -1, slot = 0, pending_n = 0;
  auto t_last = std::chrono::steady_clock::now();
  while (k < maxit) {
    const int todo = std::min(chunk, maxit - k);
    for (int i = 0; i < todo; ++i) {
      CK(c, cudaGraphLaunch(c->gexec[m], c->stream));
      c->launches += c->graph_launches_per_iter[m];
    }
    k += todo;
    CK(c, cudaMemcpyAsync(&c->done_ring[slot], &c->st->done, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaEventRecord(c->done_ev[slot], c->stream));
    if (!c->pipe) { pending = slot; pending_n = todo; }   // default: wait for this chunk
    if (pending >= 0) {
      CK(c, cudaEventSynchronize(c->done_ev[pending]));
      if (c->done_ring[pending]) { done = 1; break; }
      const auto now = std::chrono::steady_clock::now();
      const double per = std::chrono::duration<double, std::micro>(now - t_last).count() / pending_n;
      t_last = now;
      // several ranks: a schedule independent of host timing, so every rank
      // queues the same iterations (the graphs hold collectives) and all stop
      // on the same chunk (the done flag derives from allreduced scalars)
      // One rank, pipelined: the chunk queued ahead only has to cover the host
      // round trip (~25 µs), and every iteration of it is wasted (gated) work
      // once the solve has converged; unpipelined: ~200 µs per chunk.
      const double target = c->pipe ? 25.0 : 200.0;
      chunk = c->world > 1 ? std::min(32, 2 * chunk)
                           : per > 0 ? (int)std::max(1.0, std::min(32.0, std::ceil(target / per))) : 32;
    }
    pending = slot;
    pending_n = todo;
    slot ^= 1;
  }
  return CCG_OK;
}

// host-side radix-2 FFT (double) of one strided line, used once per operator
static void host_fft_line(std::complex<double>* a, int L, int64_t stride) {
  if (L <= 1) return;
  std::vector<std::complex<double>> v(L);
  int logL = 0;
  while ((1 << logL) < L) ++logL;
  for (int i = 0; i < L; ++i) {
    int r = 0;
    for (int b = 0; b < logL; ++b) r |= ((i >> b) & 1) << (logL - 1 - b);
    v[r] = a[(int64_t)i * stride];
  }
  const double PI = 3.14159265358979323846264338327950288;
  for (int h = 1; h < L; h <<= 1) {
    for (int i0 = 0; i0 < L; i0 += 2 * h)
      for (int m = 0; m < h; ++m) {
        const double ang = -PI * (double)m / (double)h;
        const std::complex<double> w(std::cos(ang), std::sin(ang));
        const std::complex<double> x0 = v[i0 + m], x1 = v[i0 + m + h] * w;
        v[i0 + m] = x0 + x1;
        v[i0 + m + h] = x0 - x1;
      }
  }
  for (int i = 0; i < L; ++i) a[(int64_t)i * stride] = v[i];
}

static int pow2_at_least(int64_t v, int* lg) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  *lg = l;
  return 1 << l;
}

template <typename T>
static int toeplitz_setup(ccg_ctx* c, const std::vector<std::complex<double>>& Kh) {
  using C = typename CT<T>::c;
  const FftGeo& g = c->geo;
  const size_t N = (size_t)g.X2 * g.Y2 * g.Z2;
  std::vector<C> kh(N);
  for (size_t i = 0; i < N; ++i) { kh[i].x = (T)Kh[i].real(); kh[i].y = (T)Kh[i].imag(); }
  const int half = std::max(1, c->fft_lmax / 2);
  std::vector<C> tw(half);
  const double PI = 3.14159265358979323846264338327950288;
  for (int k = 0; k < half; ++k) {
    const double ang = -2.0 * PI * (double)k / (double)c->fft_lmax;
    tw[k].x = (T)std::cos(ang);
    tw[k].y = (T)std::sin(ang);
  }
  CK(c, cudaMalloc(&c->fftW, N * sizeof(C)));
  CK(c, cudaMalloc(&c->fftK, N * sizeof(C)));
  CK(c, cudaMalloc(&c->fftTw, half * sizeof(C)));
  CK(c, cudaMemcpy(c->fftK, kh.data(), N * sizeof(C), cudaMemcpyHostToDevice));
  CK(c, cudaMemcpy(c->fftTw, tw.data(), half * sizeof(C), cudaMemcpyHostToDevice));
  CK(c, cudaMemset(c->fftW, 0, N * sizeof(C)));
  return CCG_OK;
}

extern "C" {

const char* ccg_version(void) { return "ccg-b200 0.1 sm_100a"; }

int ccg_get_unique_id(uint8_t id[128]) {
  if (!id) { g_create_err = "id is NULL"; return CCG_E_ARG; }
  if (!nccl_load()) { g_create_err = g_nccl.err; return CCG_E_NCCL; }
  ncclUniqueId u;
  ncclResult_t r = g_nccl.GetUniqueId(&u);
  if (r != ncclSuccess) { g_create_err = g_nccl.GetErrorString(r); return CCG_E_NCCL; }
  memcpy(id, u.internal, 128);
  return CCG_OK;
}

static int create_impl(ccg_handle* h, ccg_dtype dt, int64_t n, int world, int rank, const uint8_t* nccl_id,
                       int device, void* cuda_stream, LoopbackGroup* lg, uint32_t options = 0) {
  if (!h) { g_create_err = "h is NULL"; return CCG_E_ARG; }
  *h = nullptr;
  if (dt != CCG_C64 && dt != CCG_C128) { g_create_err = "bad dtype"; return CCG_E_ARG; }
  if (n < 1 || world < 1 || rank < 0 || rank >= world) { g_create_err = "bad n/world/rank"; return CCG_E_ARG; }
  if (n % world != 0) { g_create_err = "n must be divisible by world"; return CCG_E_DIM; }
  if (world > 1 && !nccl_id && !lg) { g_create_err = "nccl_id required for world > 1"; return CCG_E_ARG; }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    g_create_err = std::string("no CUDA device: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return CCG_E_CUDA;
  }
  if (device < 0 || device >= ndev) { g_create_err = "bad device ordinal"; return CCG_E_ARG; }
  ccg_ctx* c = new ccg_ctx();
  c->dtype = dt;
  c->esz = dt == CCG_C64 ? 8 : 16;
  c->n = n;
  c->world = world;
  c->rank = rank;
  c->mnloc = n / world;
  c->mrow0 = (int64_t)rank * c->mnloc;
  c->rep = world > 1 && (options & CCG_OPT_REPLICATED);
  c->nloc = c->rep ? n : c->mnloc;      // vectors: whole (replicated) or this rank's slice
  c->row0 = c->rep ? 0 : c->mrow0;
  c->device = device;
  {
    const char* pe = getenv("CCG_PDL");
    c->pdl = !(pe && !strcmp(pe, "0"));
  }
  auto bail = [&](int code) {
    g_create_err = c->err;
    ccg_destroy(c);
    return code;
  };
#define CKC(call)                                                                   \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      c->err = std::string(#call) + ": " + cudaGetErrorString(e_);                  \
      return bail(e_ == cudaErrorMemoryAllocation ? CCG_E_OOM : CCG_E_CUDA);        \
    }                                                                               \
  } while (0)
  CKC(cudaSetDevice(device));
  cudaDeviceProp prop;
  CKC(cudaGetDeviceProperties(&prop, device));
  c->sm_count = prop.multiProcessorCount;
  if (cuda_stream) {
    c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  } else {
    CKC(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  CKC(cudaMalloc(&c->st, sizeof(State)));
  CKC(cudaMallocHost(&c->st_host, sizeof(State)));
  CKC(cudaMallocHost(&c->done_ring, 2 * sizeof(int)));
  {
    const char* pp = getenv("CCG_PIPELINE");
    c->pipe = pp && !strcmp(pp, "1");
  }
  for (auto& e : c->done_ev) CKC(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CKC(cudaMalloc(&c->ticket, sizeof(unsigned)));
  CKC(cudaMemset(c->ticket, 0, sizeof(unsigned)));
  CKC(cudaMalloc(&c->rank_sum, 16 * sizeof(double2)));
  CKC(cudaMalloc(&c->all_sums, (size_t)16 * world * sizeof(double2)));
  CKC(cudaMalloc(&c->zero_gate, sizeof(int)));
  CKC(cudaMemset(c->zero_gate, 0, sizeof(int)));
  for (int i = 0; i < NLOCAL; ++i) {
    CKC(cudaMalloc(&c->loc[i], (size_t)c->nloc * c->esz));
    CKC(cudaMemset(c->loc[i], 0, (size_t)c->nloc * c->esz));
  }
  for (int i = 0; i < NFULL; ++i) {
    CKC(cudaMalloc(&c->full[i], (size_t)n * c->esz));
    CKC(cudaMemset(c->full[i], 0, (size_t)n * c->esz));
  }
  if (c->rep) {
    CKC(cudaMalloc(&c->rep_tmp, (size_t)n * c->esz));
    CKC(cudaMalloc(&c->rep_parts, (size_t)n * world * c->esz));
  }
  if (world > 1) {
    CKC(cudaMalloc(&c->wfull, (size_t)n * c->esz));
    if (lg) {
      {
        std::lock_guard<std::mutex> lk(lg->m);
        lg->refs++;
      }
      c->comm = new LoopbackComm(lg, rank);
    } else {
      NcclComm* nc = new NcclComm();
      c->comm = nc;
      int rc = nc->init(world, rank, nccl_id);
      if (rc) { c->err = nc->err; return bail(CCG_E_NCCL); }
    }
  }
#undef CKC
  *h = c;
  return CCG_OK;
}

int ccg_create(ccg_handle* h, ccg_dtype dt, int64_t n, int world, int rank, const uint8_t* nccl_id, int device,
               void* cuda_stream) {
  return create_impl(h, dt, n, world, rank, nccl_id, device, cuda_stream, nullptr);
}

int ccg_create_ex(ccg_handle* h, ccg_dtype dt, int64_t n, int world, int rank, const uint8_t* nccl_id, int device,
                  void* cuda_stream, uint32_t options) {
  return create_impl(h, dt, n, world, rank, nccl_id, device, cuda_stream, nullptr, options);
}

int ccg_create_loopback_group_ex(ccg_handle* hs, int world, ccg_dtype dt, int64_t n, int device, uint32_t options);
int ccg_create_loopback_group(ccg_handle* hs, int world, ccg_dtype dt, int64_t n, int device) {
  return ccg_create_loopback_group_ex(hs, world, dt, n, device, 0);
}

int ccg_create_loopback_group_ex(ccg_handle* hs, int world, ccg_dtype dt, int64_t n, int device, uint32_t options) {
  if (!hs || world < 2) { g_create_err = "hs is NULL or world < 2"; return CCG_E_ARG; }
  LoopbackGroup* lg = new LoopbackGroup(world);
  lg->refs = 1;  // held until every handle exists
  int rc = CCG_OK;
  int made = 0;
  for (int r = 0; r < world; ++r) {
    rc = create_impl(&hs[r], dt, n, world, r, nullptr, device, nullptr, lg, options);
    if (rc) break;
    made++;
  }
  if (rc) {
    for (int r = 0; r < made; ++r) ccg_destroy(hs[r]);
  }
  bool last = false;
  {
    std::lock_guard<std::mutex> lk(lg->m);
    last = (--lg->refs == 0);
  }
  if (last) delete lg;
  return rc;
}

int ccg_set_matvec_dense(ccg_handle c, const void* A_local, int64_t row0, int64_t nloc, int64_t lda, uint32_t flags) {
  if (!c) return CCG_E_ARG;
  if (!A_local) FAIL(c, CCG_E_ARG, "A_local is NULL");
  if (row0 != c->mrow0 || nloc != c->mnloc) FAIL(c, CCG_E_DIM, "row0/nloc differ from the handle's row range");
  if (lda < c->n) FAIL(c, CCG_E_DIM, "lda < n");
  if (!is_device_ptr(A_local)) FAIL(c, CCG_E_ARG, "A_local must be a device pointer");
  if (((uintptr_t)A_local) % c->esz) FAIL(c, CCG_E_ARG, "A_local misaligned");
  CK(c, cudaSetDevice(c->device));
  free_csr_copies(c);
  c->opk = OPK_DENSE;
  c->A = A_local;
  c->lda = lda;
  c->flags = flags;
  c->vec_ok = (c->esz == 16) || (((uintptr_t)A_local % 16) == 0 && (lda % 2) == 0);
  {
    // small L2-resident systems: the whole loop in one cluster (cluster.cuh)
    const char* ce = getenv("CCG_CLUSTER");
    const char* cb = getenv("CCG_CLUSTER_MAXBYTES");
    const double maxb = cb ? atof(cb) : 4.0 * 1024 * 1024;
    c->cluster_ok = c->world == 1 && !(ce && !strcmp(ce, "0")) &&
                    (double)c->n * (double)c->n * (double)c->esz <= maxb;
  }
  invalidate_graphs(c);
  return c->dtype == CCG_C64 ? choose_launch<float>(c) : choose_launch<double>(c);
}

int ccg_set_matvec_csr(ccg_handle c, const int32_t* rowptr, const int32_t* colind, const void* vals, int64_t row0,
                       int64_t nloc, int64_t nnz_local, uint32_t flags) {
  if (!c) return CCG_E_ARG;
  if (!rowptr || !colind || !vals) FAIL(c, CCG_E_ARG, "NULL CSR pointer");
  if (row0 != c->mrow0 || nloc != c->mnloc) FAIL(c, CCG_E_DIM, "row0/nloc differ from the handle's row range");
  if (nnz_local < 0 || nnz_local > INT32_MAX) FAIL(c, CCG_E_DIM, "nnz out of range");
  if (!is_device_ptr(rowptr) || !is_device_ptr(colind) || !is_device_ptr(vals))
    FAIL(c, CCG_E_ARG, "CSR arrays must be device pointers");
  CK(c, cudaSetDevice(c->device));
  // validate structure and compute the halo width on the host (one-time copy)
  std::vector<int32_t> rp(nloc + 1), ci(nnz_local);
  CK(c, cudaMemcpy(rp.data(), rowptr, (nloc + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (nnz_local) CK(c, cudaMemcpy(ci.data(), colind, nnz_local * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (rp[0] != 0 || rp[nloc] != nnz_local) FAIL(c, CCG_E_DIM, "rowptr[0] != 0 or rowptr[nloc] != nnz");
  int64_t halo = 0;
  for (int64_t i = 0; i < nloc; ++i) {
    if (rp[i + 1] < rp[i]) FAIL(c, CCG_E_ARG, "rowptr not nondecreasing");
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t j = ci[k];
      if (j < 0 || j >= c->n) FAIL(c, CCG_E_ARG, "column index out of range");
      if (j < row0) halo = std::max<int64_t>(halo, row0 - j);
      if (j >= row0 + nloc) halo = std::max<int64_t>(halo, j - (row0 + nloc) + 1);
    }
  }
  if (c->world > 1 && !c->rep && halo > nloc)
    FAIL(c, CCG_E_ARG, "CSR columns reach beyond the neighbour ranks (halo > nloc)");
  if (c->world > 1 && !c->rep) {
    // all ranks use the same (maximum) halo width so that sends match receives
    int64_t* dh = nullptr;
    CK(c, cudaMalloc(&dh, sizeof(int64_t) * c->world));
    CK(c, cudaMemcpy(dh + c->rank, &halo, sizeof(int64_t), cudaMemcpyHostToDevice));
    int r = c->comm->allgather(dh + c->rank, dh, 1, CT_I64, c->stream);
    if (r) { cudaFree(dh); FAIL(c, r, c->comm->err); }
    std::vector<int64_t> hs(c->world);
    CK(c, cudaStreamSynchronize(c->stream));
    CK(c, cudaMemcpy(hs.data(), dh, sizeof(int64_t) * c->world, cudaMemcpyDeviceToHost));
    cudaFree(dh);
    for (auto v : hs) halo = std::max(halo, v);
    if (halo > nloc) FAIL(c, CCG_E_ARG, "halo > nloc on some rank");
  }
  // CSR-stream row blocks: ≤ 256 rows and ≤ 2048 nonzeros each (long rows alone)
  free_csr_copies(c);
  const char* sp = getenv("CCG_SPMV");
  // SELL-32 copy when the padding is small (regular rows, e.g. stencils)
  {
    const int64_t nsl = (nloc + 31) / 32;
    std::vector<int64_t> off(nsl);
    std::vector<int32_t> wid(nsl);
    int64_t tot = 0;
    for (int64_t sl = 0; sl < nsl; ++sl) {
      int32_t w = 0;
      for (int64_t i = sl * 32; i < std::min<int64_t>(nloc, sl * 32 + 32); ++i) w = std::max(w, rp[i + 1] - rp[i]);
      off[sl] = tot;
      wid[sl] = w;
      tot += 32 * (int64_t)w;
    }
    const bool want = sp ? !strcmp(sp, "sell") : (tot <= nnz_local + nnz_local / 4 + 1024);
    if (want && nloc > 0) {
      CK(c, cudaMalloc(&c->sell_off, nsl * sizeof(int64_t)));
      CK(c, cudaMalloc(&c->sell_width, nsl * sizeof(int32_t)));
      CK(c, cudaMalloc(&c->sell_col, std::max<int64_t>(tot, 1) * sizeof(int32_t)));
      CK(c, cudaMalloc(&c->sell_val, std::max<int64_t>(tot, 1) * c->esz));
      CK(c, cudaMemcpy(c->sell_off, off.data(), nsl * sizeof(int64_t), cudaMemcpyHostToDevice));
      CK(c, cudaMemcpy(c->sell_width, wid.data(), nsl * sizeof(int32_t), cudaMemcpyHostToDevice));
      const int64_t thr = nsl * 32;
      const int g = (int)((thr + 255) / 256);
      if (c->esz == 8)
        csr_to_sell<float2><<<g, 256, 0, c->stream>>>(rowptr, colind, (const float2*)vals, c->sell_off,
                                                      c->sell_width, nloc, c->sell_col, (float2*)c->sell_val);
      else
        csr_to_sell<double2><<<g, 256, 0, c->stream>>>(rowptr, colind, (const double2*)vals, c->sell_off,
                                                        c->sell_width, nloc, c->sell_col, (double2*)c->sell_val);
      CK(c, cudaGetLastError());
      CK(c, cudaStreamSynchronize(c->stream));
    }
  }
  if (!c->sell_col && (sp == nullptr || strcmp(sp, "lanes") != 0)) {
    std::vector<int32_t> bl;
    bl.push_back(0);
    int64_t r = 0;
    while (r < nloc) {
      int64_t e = r + 1;
      while (e < nloc && e - r < 256 && rp[e + 1] - rp[r] <= 2048) ++e;
      bl.push_back((int32_t)e);
      r = e;
    }
    c->csr_nblocks = (int)bl.size() - 1;
    CK(c, cudaMalloc(&c->csr_blocks, bl.size() * sizeof(int32_t)));
    CK(c, cudaMemcpy(c->csr_blocks, bl.data(), bl.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  c->opk = OPK_CSR;
  c->rowptr = rowptr;
  c->colind = colind;
  c->vals = vals;
  c->nnz = nnz_local;
  c->halo = halo;
  c->flags = flags;
  c->vec_ok = true;
  invalidate_graphs(c);
  return c->dtype == CCG_C64 ? choose_launch<float>(c) : choose_launch<double>(c);
}

int ccg_set_matvec_stencil7(ccg_handle c, int64_t nx, int64_t ny, int64_t nz, const double* coeffs, uint32_t flags) {
  if (!c) return CCG_E_ARG;
  if (!coeffs) FAIL(c, CCG_E_ARG, "coeffs is NULL");
  if (nx < 1 || ny < 1 || nz < 1 || nx > INT32_MAX || ny > INT32_MAX || nz > INT32_MAX)
    FAIL(c, CCG_E_DIM, "bad lattice size");
  if (nx * ny * nz != c->n) FAIL(c, CCG_E_DIM, "nx*ny*nz != n");
  if (nz % c->world) FAIL(c, CCG_E_DIM, "nz must be divisible by world (z-slab sharding)");
  for (int i = 0; i < 8; ++i)
    if (!std::isfinite(coeffs[i])) FAIL(c, CCG_E_ARG, "non-finite stencil coefficient");
  CK(c, cudaSetDevice(c->device));
  free_csr_copies(c);
  c->opk = OPK_STENCIL;
  c->snx = (int)nx;
  c->sny = (int)ny;
  c->snz = (int)nz;
  c->snzl = (int)(nz / c->world);
  c->sz0 = c->rank * c->snzl;
  for (int i = 0; i < 4; ++i) c->scoef[i] = make_double2(coeffs[2 * i], coeffs[2 * i + 1]);
  c->halo = nx * ny;
  c->flags = flags | CCG_FLAG_SYMMETRIC;
  c->vec_ok = true;
  const char* zc = getenv("CCG_STENCIL_ZC");
  c->szc = zc ? std::max(1, atoi(zc)) : 4;
  invalidate_graphs(c);
  return c->dtype == CCG_C64 ? choose_launch<float>(c) : choose_launch<double>(c);
}

int ccg_set_matvec_toeplitz3(ccg_handle c, int64_t nx, int64_t ny, int64_t nz, const double* kernel,
                             const double* diag, uint32_t flags) {
  if (!c) return CCG_E_ARG;
  if (!kernel || !diag) FAIL(c, CCG_E_ARG, "kernel / diag is NULL");
  if (nx < 1 || ny < 1 || nz < 1 || nx > 1024 || ny > 1024 || nz > 1024)
    FAIL(c, CCG_E_DIM, "lattice sides must be in [1, 1024]");
  if (nx * ny * nz != c->n) FAIL(c, CCG_E_DIM, "nx*ny*nz != n");
  CK(c, cudaSetDevice(c->device));
  free_csr_copies(c);
  FftGeo g;
  g.nx = (int)nx; g.ny = (int)ny; g.nz = (int)nz;
  g.X2 = pow2_at_least(2 * nx - 1, &g.lx);
  g.Y2 = pow2_at_least(2 * ny - 1, &g.ly);
  g.Z2 = pow2_at_least(2 * nz - 1, &g.lz);
  const int lyz = std::max(g.Y2, g.Z2);
  // lines per CTA: at most 2048 points in shared memory, and few enough that
  // every pass launches ≥ 2 CTAs per SM (the y pass has the fewest lines)
  const int want = 2 * c->sm_count;
  g.tyz = std::max(1, std::min(g.X2, std::min(16, 2048 / lyz)));
  while (g.tyz > 1 && (g.X2 / g.tyz) * std::min(g.nz, g.Y2) < want) g.tyz >>= 1;
  g.tx = std::max(1, std::min(32, 2048 / g.X2));
  while (g.tx > 1 && (g.ny * g.nz + g.tx - 1) / g.tx < want) --g.tx;
  c->geo = g;
  c->fft_lmax = std::max(g.X2, std::max(g.Y2, g.Z2));
  // circulant embedding of the kernel, 3-D FFT in double, normalised
  const int64_t kx = 2 * nx - 1, ky = 2 * ny - 1;
  const size_t N = (size_t)g.X2 * g.Y2 * g.Z2;
  std::vector<std::complex<double>> K(N);
  auto disp = [](int m, int M, int64_t n, int64_t* d) {
    if (m < n) { *d = m; return true; }
    if (m > M - n) { *d = (int64_t)m - M; return true; }
    return false;
  };
  for (int mz = 0; mz < g.Z2; ++mz)
    for (int my = 0; my < g.Y2; ++my)
      for (int mx = 0; mx < g.X2; ++mx) {
        int64_t dx, dy, dz;
        std::complex<double> v(0.0, 0.0);
        if (disp(mx, g.X2, nx, &dx) && disp(my, g.Y2, ny, &dy) && disp(mz, g.Z2, nz, &dz) &&
            !(dx == 0 && dy == 0 && dz == 0)) {
          const int64_t ki = (dx + nx - 1) + kx * ((dy + ny - 1) + ky * (dz + nz - 1));
          v = std::complex<double>(kernel[2 * ki], kernel[2 * ki + 1]);
          if (!std::isfinite(v.real()) || !std::isfinite(v.imag())) FAIL(c, CCG_E_ARG, "non-finite kernel value");
        }
        K[((size_t)mz * g.Y2 + my) * g.X2 + mx] = v;
      }
  for (int64_t l = 0; l < (int64_t)g.Y2 * g.Z2; ++l) host_fft_line(K.data() + l * g.X2, g.X2, 1);
  for (int mz = 0; mz < g.Z2; ++mz)
    for (int mx = 0; mx < g.X2; ++mx) host_fft_line(K.data() + (size_t)mz * g.Y2 * g.X2 + mx, g.Y2, g.X2);
  for (int64_t l = 0; l < (int64_t)g.X2 * g.Y2; ++l) host_fft_line(K.data() + l, g.Z2, (int64_t)g.X2 * g.Y2);
  const double inv = 1.0 / (double)N;
  for (auto& v : K) v *= inv;
  if (!std::isfinite(diag[0]) || !std::isfinite(diag[1])) FAIL(c, CCG_E_ARG, "non-finite diagonal");
  c->tdiag = make_double2(diag[0], diag[1]);
  int rc = c->dtype == CCG_C64 ? toeplitz_setup<float>(c, K) : toeplitz_setup<double>(c, K);
  if (rc) return rc;
  c->opk = OPK_TOEPLITZ;
  c->flags = flags;
  c->vec_ok = true;
  invalidate_graphs(c);
  return c->dtype == CCG_C64 ? choose_launch<float>(c) : choose_launch<double>(c);
}

int ccg_set_matvec_callback(ccg_handle c, ccg_matvec_fn fn, void* user, uint32_t caps, uint32_t flags) {
  if (!c) return CCG_E_ARG;
  if (!fn) FAIL(c, CCG_E_ARG, "fn is NULL");
  if (!(caps & CCG_CB_A)) FAIL(c, CCG_E_ARG, "caps must include CCG_CB_A");
  CK(c, cudaSetDevice(c->device));
  free_csr_copies(c);
  CK(c, cudaMalloc(&c->cb_out, (size_t)std::max<int64_t>(c->mnloc, 1) * c->esz));
  c->opk = OPK_CALLBACK;
  c->cb_fn = fn;
  c->cb_user = user;
  c->cb_caps = caps;
  c->flags = flags;
  c->vec_ok = true;
  invalidate_graphs(c);
  return c->dtype == CCG_C64 ? choose_launch<float>(c) : choose_launch<double>(c);
}

int ccg_set_gmres_restart(ccg_handle c, int32_t m) {
  if (!c) return CCG_E_ARG;
  if (m < 1 || m > GM_MAX) FAIL(c, CCG_E_ARG, "GMRES restart length must be in [1, 64]");
  if (m != c->gm_m) invalidate_graphs(c);
  c->gm_m = m;
  return CCG_OK;
}

int ccg_set_jacobi(ccg_handle c, const void* diag_local, uint32_t flags) {
  if (!c) return CCG_E_ARG;
  (void)flags;
  CK(c, cudaSetDevice(c->device));
  invalidate_graphs(c);
  if (!diag_local) {
    if (c->jac_d) cudaFree(c->jac_d);
    if (c->jac_dinv) cudaFree(c->jac_dinv);
    if (c->jac_tmp) cudaFree(c->jac_tmp);
    c->jac_d = c->jac_dinv = c->jac_tmp = nullptr;
    return CCG_OK;
  }
  // host copy of this rank's diagonal, validated, inverted in double; the whole
  // d and 1/d are allgathered so every rank can scale whole product inputs
  const size_t es = c->esz;
  std::vector<unsigned char> hd((size_t)c->mnloc * es);
  if (is_device_ptr(diag_local)) CK(c, cudaMemcpy(hd.data(), diag_local, hd.size(), cudaMemcpyDeviceToHost));
  else memcpy(hd.data(), diag_local, hd.size());
  std::vector<unsigned char> hinv(hd.size());
  for (int64_t i = 0; i < c->mnloc; ++i) {
    double re, im;
    if (es == 8) { re = reinterpret_cast<float*>(hd.data())[2 * i]; im = reinterpret_cast<float*>(hd.data())[2 * i + 1]; }
    else { re = reinterpret_cast<double*>(hd.data())[2 * i]; im = reinterpret_cast<double*>(hd.data())[2 * i + 1]; }
    if (!(std::isfinite(re) && std::isfinite(im)) || (re == 0.0 && im == 0.0))
      FAIL(c, CCG_E_ARG, "Jacobi: diagonal entries must be finite and nonzero");
    const std::complex<double> inv = 1.0 / std::complex<double>(re, im);
    if (es == 8) {
      reinterpret_cast<float*>(hinv.data())[2 * i] = (float)inv.real();
      reinterpret_cast<float*>(hinv.data())[2 * i + 1] = (float)inv.imag();
    } else {
      reinterpret_cast<double*>(hinv.data())[2 * i] = inv.real();
      reinterpret_cast<double*>(hinv.data())[2 * i + 1] = inv.imag();
    }
  }
  const size_t full = (size_t)c->n * es;
  if (!c->jac_d) CK(c, cudaMalloc(&c->jac_d, full));
  if (!c->jac_dinv) CK(c, cudaMalloc(&c->jac_dinv, full));
  if (!c->jac_tmp) CK(c, cudaMalloc(&c->jac_tmp, full));
  CK(c, cudaMemcpy(static_cast<char*>(c->jac_d) + (size_t)c->mrow0 * es, hd.data(), hd.size(), cudaMemcpyHostToDevice));
  CK(c, cudaMemcpy(static_cast<char*>(c->jac_dinv) + (size_t)c->mrow0 * es, hinv.data(), hinv.size(),
                   cudaMemcpyHostToDevice));
  if (c->world > 1) {
    const CommType t = es == 8 ? CT_F32 : CT_F64;
    int r = c->comm->allgather_inplace(c->jac_d, (size_t)c->mnloc * 2, t, c->stream);
    if (!r) r = c->comm->allgather_inplace(c->jac_dinv, (size_t)c->mnloc * 2, t, c->stream);
    if (r) FAIL(c, r, c->comm->err);
    CK(c, cudaStreamSynchronize(c->stream));
  }
  return CCG_OK;
}

int ccg_set_bicgstab_ell(ccg_handle c, int32_t ell) {
  if (!c) return CCG_E_ARG;
  if (ell < 1 || ell > BL_MAX) FAIL(c, CCG_E_ARG, "BiCGstab(l): l must be in [1, 4]");
  if (ell != c->bl_l) invalidate_graphs(c);
  c->bl_l = ell;
  return CCG_OK;
}

static int bicgstabl_workspace(ccg_ctx* c) {
  const size_t need = (size_t)2 * (c->bl_l + 1) * (size_t)c->n * c->esz;
  if (need > c->bl_bytes) {
    if (c->bl_buf) cudaFree(c->bl_buf);
    c->bl_buf = nullptr;
    c->bl_bytes = 0;
    CK(c, cudaMalloc(&c->bl_buf, need));
    CK(c, cudaMemset(c->bl_buf, 0, need));
    c->bl_bytes = need;
  }
  invalidate_graphs(c);   // buffer layout depends on ℓ
  if (!c->gm_dev) {
    CK(c, cudaMalloc(&c->gm_dev, sizeof(GmDev)));
    CK(c, cudaMemset(c->gm_dev, 0, sizeof(GmDev)));
  }
  return CCG_OK;
}

// GMRES workspace: basis (m+1) × nloc, Hessenberg data, per-CTA multi-dot slots
static int gmres_workspace(ccg_ctx* c) {
  const size_t need = (size_t)(c->gm_m + 1) * (size_t)c->nloc * c->esz;
  if (need > c->gm_V_bytes) {
    if (c->gm_V) cudaFree(c->gm_V);
    c->gm_V = nullptr;
    c->gm_V_bytes = 0;
    CK(c, cudaMalloc(&c->gm_V, need));
    c->gm_V_bytes = need;
    invalidate_graphs(c);
  }
  if (!c->gm_dev) {   // (BiCGstab(ℓ) may have allocated the scratch already)
    CK(c, cudaMalloc(&c->gm_dev, sizeof(GmDev)));
    CK(c, cudaMemset(c->gm_dev, 0, sizeof(GmDev)));
  }
  if (!c->gm_part) {
    // one full wave of the multi-dot passes: CTAs per SM = their occupancy
    // (76-78 registers → 3 at c128; the former fixed 4 per SM left a
    // quarter of the CTAs for a second wave).  CCG_GM_CPS overrides (A/B).
    int o0 = 0, o1 = 0;
    if (c->dtype == CCG_C64) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o0, gm_pass<float, 0>, GM_NT, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, gm_pass<float, 1>, GM_NT, 0);
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o0, gm_pass<double, 0>, GM_NT, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, gm_pass<double, 1>, GM_NT, 0);
    }
    const char* gf = getenv("CCG_GM_FAST");
    c->gm_fast = !(gf && !strcmp(gf, "0"));
    if (c->gm_fast) {
      if (c->dtype == CCG_C64) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o0, gm_pass<float, 0, true>, GM_NT, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, gm_pass<float, 1, true>, GM_NT, 0);
      } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o0, gm_pass<double, 0, true>, GM_NT, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, gm_pass<double, 1, true>, GM_NT, 0);
      }
    }
    int cps = std::max(1, std::min(o0, o1));
    const char* gc = getenv("CCG_GM_CPS");
    if (gc) cps = std::max(1, std::min(32, atoi(gc)));
    c->gm_grid = (int)std::max<int64_t>(1, std::min<int64_t>((c->nloc + GM_NT - 1) / GM_NT, (int64_t)c->sm_count * cps));
    int on = 0, ox = 0;
    if (c->dtype == CCG_C64) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&on, gm_normalize<float>, 256, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ox, gm_xupdate<float>, 256, 0);
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&on, gm_normalize<double>, 256, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ox, gm_xupdate<double>, 256, 0);
    }
    c->gm_vgrid = (int)std::max<int64_t>(
        1, std::min<int64_t>((c->nloc + 255) / 256, (int64_t)c->sm_count * std::max(1, std::min(on, ox))));
    CK(c, cudaMalloc(&c->gm_part, (size_t)c->gm_grid * (GM_MAX + 1) * sizeof(double2)));
    CK(c, cudaMalloc(&c->gm_ticket, sizeof(unsigned)));
    CK(c, cudaMemset(c->gm_ticket, 0, sizeof(unsigned)));
    CK(c, cudaMalloc(&c->gm_rank, (size_t)(GM_MAX + 1) * sizeof(double2)));
    CK(c, cudaMalloc(&c->gm_all, (size_t)c->world * (GM_MAX + 1) * sizeof(double2)));
  }
  CK(c, cudaMemcpyAsync(&c->gm_dev->m, &c->gm_m, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  return CCG_OK;
}

static int stage_in(ccg_ctx* c, void* dst, const void* src, size_t bytes) {
  if (is_device_ptr(src)) {
    CK(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    CK(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
  }
  return CCG_OK;
}
static int stage_out(ccg_ctx* c, void* dst, const void* src, size_t bytes) {
  if (is_device_ptr(dst)) {
    CK(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    CK(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
  }
  return CCG_OK;
}

// user vector slices (this rank's mnloc rows) <-> library vectors; with
// replicated vectors the slice sits at mrow0 and is allgathered in place
static int vec_in(ccg_ctx* c, void* dst, const void* src) {
  const size_t bytes = (size_t)c->mnloc * c->esz;
  char* d = static_cast<char*>(dst) + (c->rep ? (size_t)c->mrow0 * c->esz : 0);
  TRY(stage_in(c, d, src, bytes));
  if (c->rep) {
    const int r = c->comm->allgather_inplace(dst, (size_t)c->mnloc * 2, c->esz == 8 ? CT_F32 : CT_F64, c->stream);
    if (r) FAIL(c, r, c->comm->err);
  }
  return CCG_OK;
}
static int vec_out(ccg_ctx* c, void* dst, const void* src) {
  const char* s = static_cast<const char*>(src) + (c->rep ? (size_t)c->mrow0 * c->esz : 0);
  return stage_out(c, dst, s, (size_t)c->mnloc * c->esz);
}

static bool needs_ah(int m) {
  return m == CCG_CGNE || m == CCG_QMR || m == CCG_BICOR || m == CCG_BICG || m == CCG_CGNR;
}

int ccg_apply(ccg_handle c, ccg_op op, const void* x_local, void* y_local) {
  if (!c) return CCG_E_ARG;
  if (!x_local || !y_local) FAIL(c, CCG_E_ARG, "NULL vector");
  if (op != CCG_OP_A && op != CCG_OP_AH && op != CCG_OP_AT) FAIL(c, CCG_E_ARG, "bad op");
  if (c->opk == OPK_NONE) FAIL(c, CCG_E_STATE, "no operator set (call ccg_set_matvec_*)");
  if (c->opk == OPK_CSR && op != CCG_OP_A && (!(c->flags & CCG_FLAG_SYMMETRIC) || (c->world > 1 && !c->rep)))
    FAIL(c, CCG_E_CAPABILITY, "CSR Aᴴ/Aᵀ needs CCG_FLAG_SYMMETRIC and world == 1 (or replicated vectors)");
  if (c->opk == OPK_CALLBACK && !(c->cb_caps & (op == CCG_OP_A ? CCG_CB_A : op == CCG_OP_AH ? CCG_CB_AH : CCG_CB_AT)))
    FAIL(c, CCG_E_CAPABILITY, "the user callback does not provide this product");
  CK(c, cudaSetDevice(c->device));
  c->launches = 0;
  c->ms_a = c->ms_ah = 0;
  c->n_a = c->n_ah = 0;
  void* xin = c->loc[3];
  void* yout = c->loc[4];
  TRY(vec_in(c, xin, x_local));
  int rc = c->dtype == CCG_C64
               ? Engine<float>::apply(c, op, (const float2*)xin, (float2*)yout)
               : Engine<double>::apply(c, op, (const double2*)xin, (double2*)yout);
  if (rc) return rc;
  TRY(vec_out(c, y_local, yout));
  CK(c, cudaStreamSynchronize(c->stream));
  tev_collect(c);
  return CCG_OK;
}

int ccg_solve(ccg_handle c, ccg_method method, const void* x0_local, const void* y_local, void* x_local_out, double tol,
              int32_t maxit, ccg_result* res) {
  auto t_start = std::chrono::steady_clock::now();
  if (!c) return CCG_E_ARG;
  if (!y_local || !x_local_out || !res) FAIL(c, CCG_E_ARG, "NULL y/x_out/res");
  if ((int)method < 0 || (int)method >= M_COUNT) FAIL(c, CCG_E_ARG, "bad method");
  if (!(tol >= 0.0) || maxit < 1) FAIL(c, CCG_E_ARG, "tol must be >= 0 and maxit >= 1");
  if (c->opk == OPK_NONE) FAIL(c, CCG_E_STATE, "no operator set (call ccg_set_matvec_*)");
  if (needs_ah(method) && c->opk == OPK_CSR && (!(c->flags & CCG_FLAG_SYMMETRIC) || (c->world > 1 && !c->rep)))
    FAIL(c, CCG_E_CAPABILITY, "method needs Aᴴ; CSR provides it only with CCG_FLAG_SYMMETRIC and world == 1");
  if (c->opk == OPK_CALLBACK && (!(c->cb_caps & CCG_CB_A) || (needs_ah(method) && !(c->cb_caps & CCG_CB_AH))))
    FAIL(c, CCG_E_CAPABILITY, "the user callback does not provide the products this method needs");
  CK(c, cudaSetDevice(c->device));
  c->launches = 0;
  c->ms_a = c->ms_ah = 0;
  c->n_a = c->n_ah = 0;
  const size_t bytes = (size_t)c->nloc * c->esz;   // library vectors (whole when replicated)
  // history buffer
  if (maxit + 1 > c->hist_cap) {
    if (c->hist) cudaFree(c->hist);
    c->hist = nullptr;
    CK(c, cudaMalloc(&c->hist, sizeof(double) * (maxit + 1)));
    c->hist_cap = maxit + 1;
  }
  // state
  State s0;
  memset(&s0, 0, sizeof(s0));
  s0.maxit = maxit;
  s0.method = method;
  s0.tol2 = tol * tol;
  s0.hist = c->hist;
  s0.hist_cap = c->hist_cap;
  if (method == CCG_GMRES) {
    TRY(gmres_workspace(c));
    s0.gm = c->gm_dev;
  }
  if (method == CCG_BICGSTABL) {
    if (c->bl_l != c->bl_built) { TRY(bicgstabl_workspace(c)); c->bl_built = c->bl_l; }
    s0.gm = c->gm_dev;
    s0.bl_l = c->bl_l;
  }
  *c->st_host = s0;
  CK(c, cudaMemcpyAsync(c->st, c->st_host, sizeof(State), cudaMemcpyHostToDevice, c->stream));
  // inputs: x -> loc[0], y -> loc[1]
  TRY(vec_in(c, c->loc[1], y_local));
  if (x0_local) {
    TRY(vec_in(c, c->loc[0], x0_local));
  } else {
    CK(c, cudaMemsetAsync(c->loc[0], 0, bytes, c->stream));
  }
  const bool has_x0 = x0_local != nullptr;
  int rc;
  if (c->jac_dinv) {
    c->jac_active = true;
    if (has_x0) {
      rc = c->dtype == CCG_C64 ? Engine<float>::jac_in(c) : Engine<double>::jac_in(c);
      if (rc) { c->jac_active = false; return rc; }
    }
  }
  if (c->opk == OPK_DENSE && c->cluster_ok && c->world == 1 && !c->timing && method != CCG_GMRES &&
      method != CCG_BICGSTABL && !c->jac_dinv) {
    // small dense system: setup, every iteration and the true residual in ONE
    // cluster launch (cluster.cuh); maxit and the stopping rule live in the State
    c->cl_method = method;
    c->cl_has_x0 = has_x0 ? 1 : 0;
    rc = c->dtype == CCG_C64 ? Engine<float>::cluster_run(c, method) : Engine<double>::cluster_run(c, method);
    if (rc) return rc;
  } else {
    rc = c->dtype == CCG_C64 ? Engine<float>::setup(c, method, has_x0) : Engine<double>::setup(c, method, has_x0);
    if (rc) return rc;
    rc = c->dtype == CCG_C64 ? run_iterations<float>(c, method, maxit) : run_iterations<double>(c, method, maxit);
    if (rc) return rc;
    rc = c->dtype == CCG_C64 ? Engine<float>::true_residual(c) : Engine<double>::true_residual(c);
    if (rc) { c->jac_active = false; return rc; }
  }
  if (c->jac_active) {
    c->jac_active = false;
    rc = c->dtype == CCG_C64 ? Engine<float>::jac_out(c) : Engine<double>::jac_out(c);
    if (rc) return rc;
  }
  CK(c, cudaMemcpyAsync(c->st_host, c->st, sizeof(State), cudaMemcpyDeviceToHost, c->stream));
  TRY(vec_out(c, x_local_out, c->loc[0]));
  CK(c, cudaStreamSynchronize(c->stream));
  tev_collect(c);
  const State& s = *c->st_host;
  memset(res, 0, sizeof(*res));
  res->status = s.done ? s.status : CCG_MAXIT;
  res->iterations = s.done ? s.iterations : maxit;
  res->matvecs_a = s.matvecs_a + (has_x0 ? 1 : 0);
  res->matvecs_ah = s.matvecs_ah;
  res->breakdown_code = s.breakdown;
  res->half_step = s.half;
  const double r0 = sqrt(s.r0sq);
  res->rec_rel_res = r0 > 0 ? sqrt(s.rr) / r0 : 0.0;
  res->true_rel_res = r0 > 0 ? sqrt(s.true_rr) / r0 : 0.0;
  if (!std::isfinite(s.true_rr)) res->status = CCG_NONFINITE;
  if (res->status == CCG_CONVERGED && res->true_rel_res > 10.0 * tol) res->status = CCG_FALSE_CONVERGENCE;
  if (c->timing) {
    // average over EXECUTED products: launches gated off after convergence
    // (e.g. CGNE's Aᴴr in the converged iteration) return at once and would
    // otherwise deflate the per-launch time (their few µs stay in the sum)
    c->n_a = std::min(c->n_a, res->matvecs_a + 1);   // + the true-residual product
    c->n_ah = std::min(c->n_ah, res->matvecs_ah);
  }
  c->hist_len = std::min(c->hist_cap, res->iterations + 1);
  res->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  return CCG_OK;
}

int ccg_get_history(ccg_handle c, double* rel_res, int32_t cap, int32_t* len) {
  if (!c || !len) return CCG_E_ARG;
  if (!c->hist || c->hist_len == 0) { *len = 0; return CCG_OK; }
  int32_t m = std::min<int32_t>(cap, c->hist_len);
  if (m > 0 && rel_res) CK(c, cudaMemcpy(rel_res, c->hist, sizeof(double) * m, cudaMemcpyDeviceToHost));
  *len = m;
  return CCG_OK;
}

int ccg_set_timing(ccg_handle c, int enable) {
  if (!c) return CCG_E_ARG;
  c->timing = enable != 0;
  return CCG_OK;
}

int ccg_get_timing(ccg_handle c, double* ms_a, int32_t* n_a, double* ms_ah, int32_t* n_ah) {
  if (!c) return CCG_E_ARG;
  if (ms_a) *ms_a = c->ms_a;
  if (n_a) *n_a = c->n_a;
  if (ms_ah) *ms_ah = c->ms_ah;
  if (n_ah) *n_ah = c->n_ah;
  return CCG_OK;
}

int64_t ccg_last_launch_count(ccg_handle c) { return c ? c->launches : -1; }

void* ccg_get_stream(ccg_handle c) { return c ? (void*)c->stream : nullptr; }

const char* ccg_last_error(ccg_handle c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int ccg_destroy(ccg_handle c) {
  if (!c) return CCG_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  invalidate_graphs(c);
  for (auto e : c->ev) cudaEventDestroy(e);
  for (auto e : c->done_ev) if (e) cudaEventDestroy(e);
  if (c->done_ring) cudaFreeHost(c->done_ring);
  delete c->comm;
  c->comm = nullptr;
  for (int i = 0; i < NLOCAL; ++i) if (c->loc[i]) cudaFree(c->loc[i]);
  for (int i = 0; i < NFULL; ++i) if (c->full[i]) cudaFree(c->full[i]);
  if (c->wfull) cudaFree(c->wfull);
  if (c->rep_tmp) cudaFree(c->rep_tmp);
  if (c->rep_parts) cudaFree(c->rep_parts);
  if (c->hpart) cudaFree(c->hpart);
  if (c->npart) cudaFree(c->npart);
  free_csr_copies(c);
  if (c->part) cudaFree(c->part);
  if (c->hist) cudaFree(c->hist);
  if (c->gm_V) cudaFree(c->gm_V);
  if (c->bl_buf) cudaFree(c->bl_buf);
  if (c->jac_d) cudaFree(c->jac_d);
  if (c->jac_dinv) cudaFree(c->jac_dinv);
  if (c->jac_tmp) cudaFree(c->jac_tmp);
  if (c->gm_dev) cudaFree(c->gm_dev);
  if (c->gm_part) cudaFree(c->gm_part);
  if (c->gm_ticket) cudaFree(c->gm_ticket);
  if (c->gm_rank) cudaFree(c->gm_rank);
  if (c->gm_all) cudaFree(c->gm_all);
  if (c->st) cudaFree(c->st);
  if (c->st_host) cudaFreeHost(c->st_host);
  if (c->ticket) cudaFree(c->ticket);
  if (c->rank_sum) cudaFree(c->rank_sum);
  if (c->all_sums) cudaFree(c->all_sums);
  if (c->zero_gate) cudaFree(c->zero_gate);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return CCG_OK;
}

}  // extern "C"
