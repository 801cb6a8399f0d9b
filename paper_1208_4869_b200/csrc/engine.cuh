// engine.cuh — the handle (ccg_ctx) and Engine<T>: kernel launches of the
// matvec engine, the collectives around them and the per-method iteration
// schedules (declared here; defined in the methods_*.cu translation units,
// compiled once per dtype so libccg.so builds in parallel).  The C-ABI is
// ccg.cu.
//
// Paper mapping (PAPER.md = P:<line>):  matvec / cmatvec separated from the
// iteration (P:17, P:95 [§5]) -> ccg_set_matvec_* + the kernels of
// matvec.cuh; cgmodule's epsilon_err / maxit -> ccg_solve(tol, maxit);
// ddprecision.f90 single/double switch -> ccg_dtype.
#pragma once
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
#include "p2p.cuh"

#include <complex>
#include <unordered_map>

using namespace ccg;


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
  // P2P mirror exchange (CCG_OPT_P2P, p2p.cuh): rep_tmp / rep_parts live in a
  // double-buffered mirror region [parity][rep_tmp n | rep_parts world·n] +
  // flags, which every rank's product epilogue writes directly
  bool p2p = false;
  void* mirror = nullptr;               // this rank's region (owned)
  size_t mirror_bytes = 0, mirror_half = 0;   // bytes; offset of parity 1
  size_t mirror_flags = 0;              // offset of the flag array (P2P_MAX uint64)
  char* peer_base[P2P_MAX] = {};        // every rank's region (this process's addresses)
  ncclWindow_t win = nullptr;           // NCCL symmetric-memory window (NCCL mode)
  uint64_t* p2p_ctr = nullptr;          // device: send / receive epochs
  int world = 1, rank = 0, device = 0;
  bool dist = false;                    // sharded code path with a communicator (world > 1, or
                                        // CCG_OPT_FORCE_COMM: a one-rank NCCL communicator)
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
  int snx = 0, sny = 0, snz = 0, sz0 = 0, snzl = 0, szc = 8;
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
  int bs_fuse = 1;        // BiCGSTAB P/S passes folded into the products (Engine::in_fuse_ok; CCG_BS_FUSE)
  int bs_merge = 0;       // BiCGSTAB X and P passes merged on the stencil / SELL SpMV (Engine::bs_merge_ok; CCG_BS_MERGE)
  int bs_fuse_ro = 0;     // the S fold on the stencil / SELL SpMV (Engine::in_fuse_ro_ok; CCG_BS_FUSE_RO)
  int split_fuse = 0;     // several strips: strip sum + epilogue by the last CTA of each row block (CCG_SPLIT_FUSE)
  unsigned* rb_ticket = nullptr;   // [split_nrb] arrival tickets (zero between launches)
  int rb_ticket_cap = 0;
  bool cols_ok = false;   // column-owner GEMV usable (vectorised layout, n % V == 0)
  int cols_strips = 1, cols_S = 1, dual_S = 1, cols_rg = 1;
  bool qmr_dual = true;   // QMR: A·p and Aᴴ·q in one pass over A (env CCG_QMR_DUAL=0 disables)
  int l2_pin = 0;         // rows ((i>>3)&63) < l2_pin of A are kept L2-resident during a solve (CCG_L2_PIN_MB)
  bool pin_on = false;    // inside ccg_solve (dense operator)
  void* npart = nullptr;  // [strips][nloc] partial row sums of the split / column-owner GEMV
  size_t npart_bytes = 0;
  // complex-symmetric dense A (CCG_FLAG_SYMMETRIC, one rank): upper-triangle
  // products (matvec.cuh gemv_sym; CCG_SYMV=0 disables)
  bool dual_rows = false; int dual_H = 512;   // QMR/BiCG dual product in the warp-per-row layout (CCG_DUAL_ROWS)
  bool cl_redundant = true;  // cluster BiCGSTAB with redundant all-row passes (3 barriers/it; CCG_CL_REDUNDANT)
  bool fft_yz = false;     // FFT lattice operator: passes 2-4 fused (fft.cuh fft_yz; CCG_FFT_YZ)
  int stencil_minb = 4;   // stencil7_kernel launch bound: 4 CTAs/SM (≤ 64 registers); CCG_STENCIL_MINB=1: none
  bool stencil_realo = true;   // skip the FMAs by exactly-zero imaginary parts of ox, oy, oz (CCG_STENCIL_REALO=0: keep them)
  bool sym_ok = false;
  int sym_state = 0;      // 0 general, 1 declared (CCG_FLAG_SYMMETRIC), 2 detected (A = Aᵀ bitwise)
  int sym_H = 64, sym_ntiles = 0, sym_strips = 1, sym_s2_grid = 1;
  int2* sym_tiles = nullptr;
  int sym2_H = 64, sym2_ntiles = 0, sym2_strips = 1;   // the dual product's tiles (gemv_sym_dual)
  int2* sym2_tiles = nullptr;
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
  // ccg_get_stat: what the last solve executed (collectives: host-side calls;
  // a call captured in the iteration graph counts once per replay)
  int64_t coll_per_iter[M_COUNT] = {};
  int64_t stat_replays = 0, stat_graph_coll = 0, stat_eager_coll = 0, stat_capture_calls = 0;
  int64_t p2p_calls = 0;   // P2P mirror exchanges issued (host side; a captured one counts once)
  bool capturing = false;
  bool pdl = true;        // programmatic dependent launch (env CCG_PDL=0 disables)
  std::unordered_map<const void*, int> occ_cache;   // per-kernel occupancy / attribute flags (this device)
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

// internal (never returned through the C-ABI): the single-cluster solve is not
// available on this device; the caller takes the graph path
enum { CCG_FALLBACK = 1000 };

#define TRY(expr)            \
  do {                       \
    int rc_ = (expr);        \
    if (rc_ != CCG_OK) return rc_; \
  } while (0)

template <typename... KArgs, typename... Args>
static void launch_k(ccg_ctx* c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  if (smem > 48 * 1024) {   // opt-in dynamic shared memory, once per kernel and handle (device)
    int& big = c->occ_cache[reinterpret_cast<const void*>(kern)];
    if (!(big & 2)) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      big |= 2;
    }
  }
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

// setup copy from (pageable) host memory, ordered on the handle's stream: the
// consumers run on c->stream (non-blocking), which a legacy-stream cudaMemcpy
// would not order against; synchronised so `src` may be freed on return
static int h2d(ccg_ctx* c, void* dst, const void* src, size_t bytes) {
  CK(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return CCG_OK;
}

static Red make_red(ccg_ctx* c) {
  Red r;
  r.part = c->part;
  r.ticket = c->ticket;
  r.rank_sum = c->rank_sum;
  r.fuse = (!c->dist || c->rep) ? 1 : 0;   // replicated vectors: reductions are local
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
  // L2-resident rows of A (matvec.cuh): only inside ccg_solve
  static int pin(const ccg_ctx* c) { return c->pin_on ? c->l2_pin : 0; }

  // -------------------- collectives --------------------
  static int allgather(ccg_ctx* c, int fi) {
    if (!c->dist || c->rep) return CCG_OK;   // replicated vectors are whole on every rank
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
      if (c->dist && !c->rep) {
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
    int& occ = c->occ_cache[reinterpret_cast<const void*>(pass_kernel<NT, Op>)];   // per handle (device)
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
          make_red(c), c->st, gate, XLoad<T>{});
    }
    else if (c->csr_blocks)
      launch_k(c, spmv_stream_kernel<T, NT, SNNZ, CONJ, Epi>, c->spmv_grid, NT, 0, c->stream, 
          c->rowptr, c->colind, vals, x, c->csr_blocks, c->csr_nblocks, epi, make_red(c), c->st, gate);
    else
      launch_k(c, spmv_csr_kernel<T, LPR, NT, CONJ, Epi>, c->spmv_grid, NT, 0, c->stream, 
          c->rowptr, c->colind, vals, x, c->mnloc, epi, make_red(c), c->st, gate);
  }

  // does this kernel use more than a few words of local memory per thread (register spills)?  Asked once
  // per kernel and handle; bits 4 (asked) and 8 (yes) of the handle's per-kernel flags
  static bool kernel_spills(ccg_ctx* c, const void* kern) {
    int& f = c->occ_cache[kern];
    if (!(f & 4)) {
      cudaFuncAttributes a;
      f |= 4;
      if (cudaFuncGetAttributes(&a, kern) == cudaSuccess && a.localSizeBytes > 96) f |= 8;
    }
    return (f & 8) != 0;
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
    // real off-diagonal coefficients (config 5's Laplacian): half the FMAs per neighbour term
    const bool realo = c->stencil_realo && k[1].y == (T)0 && k[2].y == (T)0 && k[3].y == (T)0;
    // the epilogue's early load is this product's own input (BsT, CrAr): the variant without it
    bool prex = false;
    if constexpr (EpiPreSrc<Epi>::has)
      prex = EpiPreSrc<Epi>::get(epi) == static_cast<const void*>(xfull + (int64_t)c->sz0 * c->snx * c->sny);
    auto kern = stencil7_kernel<T, Epi, XLoad<T>, 1, false>;
    if (c->stencil_minb == 3 && realo) {   // CCG_STENCIL_MINB=3: every epilogue at 3 CTAs/SM (A/B)
      kern = stencil7_kernel<T, Epi, XLoad<T>, 3, true>;
      if constexpr (EpiPreSrc<Epi>::has) { if (prex) kern = stencil7_kernel<T, Epi, XLoad<T>, 3, true, true>; }
    } else if (c->stencil_minb >= 3) {
      if (realo) {
        // 4 CTAs/SM (64 registers) unless the epilogue then spills (TFQMR's TfO: 256 B, CGS's CsR: 128 B
        // of local memory per thread; the others ≤ 32) — those run at 3 CTAs/SM (80 registers, no spills)
        kern = stencil7_kernel<T, Epi, XLoad<T>, 4, true>;
        if constexpr (EpiPreSrc<Epi>::has) { if (prex) kern = stencil7_kernel<T, Epi, XLoad<T>, 4, true, true>; }
        if (kernel_spills(c, reinterpret_cast<const void*>(kern))) kern = stencil7_kernel<T, Epi, XLoad<T>, 3, true>;
      } else {
        kern = stencil7_kernel<T, Epi, XLoad<T>, 3, false>;
        if constexpr (EpiPreSrc<Epi>::has) { if (prex) kern = stencil7_kernel<T, Epi, XLoad<T>, 3, false, true>; }
      }
    }
    launch_k(c, kern, g, 256, 0, c->stream, xfull, c->snx, c->sny, c->snz, c->sz0, c->snzl, c->szc,
                                                       k[0], k[1], k[2], k[3], epi, make_red(c), c->st, gate, XLoad<T>{});
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
    if (c->fft_yz) {   // passes 2-4 in one kernel: one kx plane per CTA in shared memory
      const size_t smp = (size_t)g.Y2 * (g.Z2 + 1) * sizeof(C);
      auto k = op == 0 ? fft_yz<T, false> : fft_yz<T, true>;
      int& attr = c->occ_cache[reinterpret_cast<const void*>(k)];
      if (!attr) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp);
        attr = 1;
      }
      launch_k(c, k, g.X2, 512, smp, c->stream, W, Kh, g, tw, L / g.Y2, L / g.Z2, gate);
      c->launches -= 2;
    } else {
      launch_k(c, fft_fwd_y<T>, dim3(g.X2 / g.tyz, g.nz), bty, smy, c->stream, W, g, tw, L / g.Y2, gate);
      if (op == 0)
        launch_k(c, fft_z_mul<T, false>, dim3(g.X2 / g.tyz, g.Y2), btz, smz, c->stream, W, Kh, g, tw, L / g.Z2, gate);
      else
        launch_k(c, fft_z_mul<T, true>, dim3(g.X2 / g.tyz, g.Y2), btz, smz, c->stream, W, Kh, g, tw, L / g.Z2, gate);
      launch_k(c, fft_inv_y<T>, dim3(g.X2 / g.tyz, g.nz), bty, smy, c->stream, W, g, tw, L / g.Y2, gate);
    }
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
    if (c->p2p) {   // rows already mirrored into every rank by the product epilogue
      TRY(p2p_exchange(c, gate));
      EpiPassMirror<T, Epi> ep{epi, mirror_view(c, 0)};
      return pass(c, ep, gate);
    }
    C* tmp = reinterpret_cast<C*>(c->rep_tmp);
    NK(c, c->comm->allgather_inplace(tmp, (size_t)c->mnloc * 2, ndt(), c->stream));
    EpiPass<C, Epi> ep{epi, tmp};
    return pass(c, ep, gate);
  }

  // -------------------- P2P mirror exchange (p2p.cuh) --------------------
  // the product epilogue: element i of this rank's output -> element off + i of
  // every rank's mirror buffer `which` (0 = rep_tmp, 1 = rep_parts)
  static MirrorStore<T> mirror_store(ccg_ctx* c, int which, int64_t off) {
    MirrorStore<T> m{};
    const size_t base = which == 0 ? 0 : (size_t)c->n * sizeof(C);
    for (int par = 0; par < 2; ++par)
      for (int p = 0; p < c->world; ++p)
        m.dst[par][p] = reinterpret_cast<C*>(c->peer_base[p] + par * c->mirror_half + base) + off;
    m.ctr = c->p2p_ctr;
    m.world = c->world;
    return m;
  }
  static MirrorView<T> mirror_view(ccg_ctx* c, int which) {
    MirrorView<T> v{};
    const size_t base = which == 0 ? 0 : (size_t)c->n * sizeof(C);
    for (int par = 0; par < 2; ++par)
      v.buf[par] = reinterpret_cast<const C*>(static_cast<char*>(c->mirror) + par * c->mirror_half + base);
    v.ctr = c->p2p_ctr;
    return v;
  }
  // after the mirrored product: publish this rank's epoch, (loopback: host
  // barrier), wait for every rank's
  static int p2p_exchange(ccg_ctx* c, const int* gate) {
    P2pCtl ctl{};
    for (int p = 0; p < c->world; ++p)
      ctl.flags[p] = reinterpret_cast<uint64_t*>(c->peer_base[p] + c->mirror_flags);
    ctl.ctr = c->p2p_ctr;
    ctl.world = c->world;
    ctl.rank = c->rank;
    launch_k(c, p2p_signal, 1, 1, 0, c->stream, ctl, gate);
    CK(c, cudaGetLastError());
    NK(c, c->comm->sync_point(c->stream));
    launch_k(c, p2p_wait, 1, 1, 0, c->stream, ctl, gate);
    c->launches += 2;
    c->p2p_calls++;
    CK(c, cudaGetLastError());
    return CCG_OK;
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
      if (c->p2p) TRY(matvec_rows(c, xfull, mirror_store(c, 0, c->mrow0), gate));
      else TRY(matvec_rows(c, xfull, Store<T>{reinterpret_cast<C*>(c->rep_tmp) + c->mrow0}, gate));
      return rep_finish_rows(c, epi, gate);
    }
    return matvec_rows(c, xfull, epi, gate);
  }

  // the input transforms of matvec_a_in apply: single GPU, dense split GEMV
  // with several strips and the strip sum in its own kernel (the epilogue that
  // rewrites the transformed vectors runs after every CTA has staged them)
  static bool in_fuse_ok(const ccg_ctx* c) {
    if (c->bs_fuse && c->opk == OPK_DENSE && c->sym_ok && !c->dist && !c->jac_active) return true;   // gemv_sym
    return c->bs_fuse && c->opk == OPK_DENSE && !c->sym_ok && c->gemv_mode == GEMV_SPLIT && c->split_strips > 1 &&
           !c->split_fuse && !c->dist && !c->jac_active;
  }
  // input transforms that read only vectors the product does not write
  // (BiCGSTAB's s = r − αv): also the stencil and the SELL SpMV, whose
  // neighbouring CTAs read the same inputs — single GPU (no halo of r, v)
  static bool in_fuse_ro_ok(const ccg_ctx* c) {
    if (in_fuse_ok(c)) return true;
    return c->bs_fuse_ro && !c->dist && !c->jac_active &&
           (c->opk == OPK_STENCIL || (c->opk == OPK_CSR && c->sell_col));
  }

  // BiCGSTAB with the X and P passes merged (methods.cuh BsTm / BsXP): single GPU, sparse operators
  static bool bs_merge_ok(const ccg_ctx* c) {
    return c->bs_merge && !c->dist && !c->jac_active && !c->bs_fuse_ro &&
           (c->opk == OPK_STENCIL || (c->opk == OPK_CSR && c->sell_col));
  }

  // y = A·x with x_j = xin(j) formed while the split GEMV stages its strips
  // (or, for in_fuse_ro_ok transforms, while the stencil / SELL SpMV loads it)
  template <class XIn, class Epi>
  static int matvec_a_in(ccg_ctx* c, XIn xin, Epi epi, const int* gate) {
    if (c->opk == OPK_STENCIL || c->opk == OPK_CSR) {
      tev_begin(c, 0);
      if (c->opk == OPK_STENCIL) {
        C k[4];
        for (int i = 0; i < 4; ++i) { k[i].x = (T)c->scoef[i].x; k[i].y = (T)c->scoef[i].y; }
        dim3 g((c->snx + 31) / 32, (c->sny + 7) / 8, (c->snzl + c->szc - 1) / c->szc);
        launch_k(c, stencil7_kernel<T, Epi, XIn>, g, 256, 0, c->stream, static_cast<const C*>(nullptr), c->snx,
                 c->sny, c->snz, c->sz0, c->snzl, c->szc, k[0], k[1], k[2], k[3], epi, make_red(c), c->st, gate, xin);
      } else {
        auto k = c->sell_one ? spmv_sell_kernel<T, NT, false, true, Epi, XIn>
                             : spmv_sell_kernel<T, NT, false, false, Epi, XIn>;
        launch_k(c, k, c->sell_grid[c->sell_one], NT, 0, c->stream, c->sell_off, c->sell_width, c->sell_col,
                 reinterpret_cast<const C*>(c->sell_val), static_cast<const C*>(nullptr), c->mnloc, epi, make_red(c),
                 c->st, gate, xin);
      }
      c->launches++;
      tev_end(c);
      CK(c, cudaGetLastError());
      return CCG_OK;
    }
    if (c->opk == OPK_DENSE && c->sym_ok) {   // upper-triangle product, x staged through xin
      tev_begin(c, 0);
      sym_product(c, static_cast<const C*>(nullptr), false, epi, gate, xin);
      c->launches += 2;
      tev_end(c);
      CK(c, cudaGetLastError());
      return CCG_OK;
    }
    const C* A = reinterpret_cast<const C*>(c->A);
    C* part = reinterpret_cast<C*>(c->npart);
    dim3 g(c->split_strips, c->split_nrb);
    const size_t smem = (size_t)c->split_W * sizeof(C);
    Store<T> none{nullptr};
    tev_begin(c, 0);
    if (c->vec_ok)
      launch_k(c, gemv_n_split<T, NT, SUR, true, false, Store<T>, XIn>, g, NT, smem, c->stream, A, c->lda,
               static_cast<const C*>(nullptr), c->n, c->mnloc, c->split_W, part, none, make_red(c), c->st, gate, pin(c),
               c->rb_ticket, xin);
    else
      launch_k(c, gemv_n_split<T, NT, SUR, false, false, Store<T>, XIn>, g, NT, smem, c->stream, A, c->lda,
               static_cast<const C*>(nullptr), c->n, c->mnloc, c->split_W, part, none, make_red(c), c->st, gate, pin(c),
               c->rb_ticket, xin);
    c->launches++;
    CK(c, cudaGetLastError());
    launch_k(c, gemv_h_stage2<T, NT, Epi>, c->nstage2_grid, NT, 0, c->stream, part, c->split_strips, c->mnloc, 0,
             c->mnloc, epi, make_red(c), c->st, gate);
    c->launches++;
    tev_end(c);
    CK(c, cudaGetLastError());
    return CCG_OK;
  }

  // complex-symmetric dense product from the upper triangle (gemv_sym):
  // conj => Aᴴx = conj(A)·x; Aᵀ = A
  template <class Epi, class XIn = XLoad<T>>
  static void sym_product(ccg_ctx* c, const C* x, bool conj, Epi epi, const int* gate, XIn xin = XIn{}) {
    const C* A = reinterpret_cast<const C*>(c->A);
    C* np = reinterpret_cast<C*>(c->npart);
    C* hp = reinterpret_cast<C*>(c->hpart);
    const State* stc = c->st;
    if (conj)
      launch_k(c, gemv_sym<T, NT, true, XIn>, c->sym_ntiles, NT, 0, c->stream, A, c->lda, x, c->n, c->sym_H,
               static_cast<const int2*>(c->sym_tiles), np, hp, gate, pin(c), stc, xin);
    else
      launch_k(c, gemv_sym<T, NT, false, XIn>, c->sym_ntiles, NT, 0, c->stream, A, c->lda, x, c->n, c->sym_H,
               static_cast<const int2*>(c->sym_tiles), np, hp, gate, pin(c), stc, xin);
    launch_k(c, gemv_sym_stage2<T, NT, Epi>, c->sym_s2_grid, NT, 0, c->stream, static_cast<const C*>(np),
             static_cast<const C*>(hp), c->n, c->sym_H, NT * CT<T>::V, c->sym_strips, epi, make_red(c), c->st, gate);
  }

  // this rank's rows of A·x (all operators), epilogue per row
  template <class Epi>
  static int matvec_rows(ccg_ctx* c, const C* xfull, Epi epi, const int* gate) {
    tev_begin(c, 0);
    if (c->opk == OPK_TOEPLITZ) {
      toeplitz(c, xfull, 0, epi, gate);
    } else if (c->opk == OPK_STENCIL) {
      stencil(c, xfull, false, epi, gate);
    } else if (c->opk == OPK_DENSE && c->sym_ok) {
      sym_product(c, xfull, false, epi, gate);
      c->launches++;   // + the stage-2 launch counted below
    } else if (c->opk == OPK_DENSE && c->gemv_mode == GEMV_SPLIT) {
      const C* A = reinterpret_cast<const C*>(c->A);
      C* part = reinterpret_cast<C*>(c->npart);
      dim3 g(c->split_strips, c->split_nrb);
      const size_t smem = (size_t)c->split_W * sizeof(C);
      if (c->split_strips == 1 || c->split_fuse) {   // epilogue in the GEMV (last strip CTA per row block)
        if (c->vec_ok)
          launch_k(c, gemv_n_split<T, NT, SUR, true, true, Epi>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, epi, make_red(c), c->st, gate, pin(c), c->rb_ticket, XLoad<T>{});
        else
          launch_k(c, gemv_n_split<T, NT, SUR, false, true, Epi>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, epi, make_red(c), c->st, gate, pin(c), c->rb_ticket, XLoad<T>{});
      } else {
        Store<T> none{nullptr};
        if (c->vec_ok && c->split_ur == 16)
          launch_k(c, gemv_n_split<T, NT, 16, true, false, Store<T>>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, none, make_red(c), c->st, gate, pin(c), c->rb_ticket, XLoad<T>{});
        else if (c->vec_ok && c->split_ur == 4)
          launch_k(c, gemv_n_split<T, NT, 4, true, false, Store<T>>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, none, make_red(c), c->st, gate, pin(c), c->rb_ticket, XLoad<T>{});
        else if (c->vec_ok)
          launch_k(c, gemv_n_split<T, NT, SUR, true, false, Store<T>>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, none, make_red(c), c->st, gate, pin(c), c->rb_ticket, XLoad<T>{});
        else
          launch_k(c, gemv_n_split<T, NT, SUR, false, false, Store<T>>, g, NT, smem, c->stream, 
              A, c->lda, xfull, c->n, c->mnloc, c->split_W, part, none, make_red(c), c->st, gate, pin(c), c->rb_ticket, XLoad<T>{});
        c->launches++;
        CK(c, cudaGetLastError());
        launch_k(c, gemv_h_stage2<T, NT, Epi>, c->nstage2_grid, NT, 0, c->stream, part, c->split_strips, c->mnloc, 0,
                                                                          c->mnloc, epi, make_red(c), c->st, gate);
      }
    } else if (c->opk == OPK_DENSE && c->gemv_mode == GEMV_COLS && c->cols_ok) {
      C* part = reinterpret_cast<C*>(c->npart);
      if (c->cols_rg == 4)
        launch_k(c, gemv_cols<T, NT, true, false, false, 4>, dim3(c->cols_strips, c->cols_S), NT, 0, c->stream, 
            reinterpret_cast<const C*>(c->A), c->lda, xfull, nullptr, c->mnloc, c->n, part, nullptr, gate, pin(c));
      else
        launch_k(c, gemv_cols<T, NT, true, false, false, 1>, dim3(c->cols_strips, c->cols_S), NT, 0, c->stream, 
            reinterpret_cast<const C*>(c->A), c->lda, xfull, nullptr, c->mnloc, c->n, part, nullptr, gate, pin(c));
      c->launches++;
      CK(c, cudaGetLastError());
      launch_k(c, gemv_h_stage2<T, NT, Epi>, c->nstage2_grid, NT, 0, c->stream, part, c->cols_strips, c->mnloc, 0, c->mnloc,
                                                                        epi, make_red(c), c->st, gate);
    } else if (c->opk == OPK_DENSE && c->gemv_mode == GEMV_BULK && c->bulk_ok) {
      constexpr size_t smem = bulk_smem_bytes<BR, BSTAGES>();
      auto kern = gemv_n_bulk<T, BR, BSTAGES, Epi>;
      int& attr_set = c->occ_cache[reinterpret_cast<const void*>(kern)];   // per handle (device)
      if (!attr_set) {
        CK(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set = 1;
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
    const bool gathered_in = c->dist && !c->rep;   // the input needs gathering first
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
      if (c->rep && c->p2p) launch(mirror_store(c, 0, c->mrow0));
      else if (c->rep) launch(Store<T>{reinterpret_cast<C*>(c->rep_tmp) + c->mrow0});
      else launch(epi);
      c->launches++;
      tev_end(c);
      CK(c, cudaGetLastError());
      if (c->rep) return rep_finish_rows(c, epi, gate);
      return post<Epi>(c, gate);
    }
    if (c->sym_ok) {   // one rank, A = Aᵀ: Aᵀx = A·x, Aᴴx = conj(A)·x from the upper triangle
      tev_begin(c, 1);
      sym_product(c, xloc, conj, epi, gate);
      c->launches += 2;
      tev_end(c);
      CK(c, cudaGetLastError());
      return CCG_OK;
    }
    const C* A = reinterpret_cast<const C*>(c->A);
    C* part = reinterpret_cast<C*>(c->hpart);
    const C* xr = c->rep ? xloc + c->mrow0 : xloc;   // the x entries of this rank's rows
    dim3 g1(c->ah_strips, c->ah_S);
    tev_begin(c, 1);
    if (c->vec_ok) {
      if (conj)
        launch_k(c, gemv_h_stage1<T, true, NT, UR, true>, g1, NT, 0, c->stream, A, c->lda, xr, c->mnloc, c->n, part, gate, pin(c));
      else
        launch_k(c, gemv_h_stage1<T, false, NT, UR, true>, g1, NT, 0, c->stream, A, c->lda, xr, c->mnloc, c->n, part, gate, pin(c));
    } else {
      if (conj)
        launch_k(c, gemv_h_stage1<T, true, NT, UR, false>, g1, NT, 0, c->stream, A, c->lda, xr, c->mnloc, c->n, part, gate, pin(c));
      else
        launch_k(c, gemv_h_stage1<T, false, NT, UR, false>, g1, NT, 0, c->stream, A, c->lda, xr, c->mnloc, c->n, part, gate, pin(c));
    }
    c->launches++;
    CK(c, cudaGetLastError());
    if (!c->dist) {
      launch_k(c, gemv_h_stage2<T, NT, Epi>, c->stage2_grid, NT, 0, c->stream, part, c->ah_S, c->n, 0, c->n, epi,
                                                                       make_red(c), c->st, gate);
      c->launches++;
      tev_end(c);
      CK(c, cudaGetLastError());
      return CCG_OK;
    }
    // multi GPU: full-length partial of this rank
    if (c->rep && c->p2p) {   // straight into slot `rank` of every rank's partial array
      launch_k(c, gemv_h_stage2<T, NT, MirrorStore<T>>, c->stage2_grid, NT, 0, c->stream, part, c->ah_S, c->n, 0, c->n,
               mirror_store(c, 1, (int64_t)c->rank * c->n), make_red(c), c->st, gate);
      c->launches++;
      tev_end(c);
      CK(c, cudaGetLastError());
      TRY(p2p_exchange(c, gate));
      EpiPassMirrorSum<T, Epi> ep{epi, mirror_view(c, 1), c->world, c->n};
      return pass(c, ep, gate);
    }
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
    if (c->sym_ok) {   // complex-symmetric A: both products from one upper-triangle pass
      const int64_t ns = (int64_t)c->sym2_strips * c->n, nh = (int64_t)((c->n + c->sym2_H - 1) / c->sym2_H) * c->n;
      const int CW2 = 128 * CT<T>::V;
      tev_begin(c, 0);
      launch_k(c, gemv_sym_dual<T, NT>, c->sym2_ntiles, NT, 0, c->stream, A, c->lda, pfull, qloc, c->n, c->sym2_H,
               static_cast<const int2*>(c->sym2_tiles), np, hp, np + ns, hp + nh, gate);
      launch_k(c, gemv_sym_stage2<T, NT, EpiA>, c->sym_s2_grid, NT, 0, c->stream, static_cast<const C*>(np),
               static_cast<const C*>(hp), c->n, c->sym2_H, CW2, c->sym2_strips, ea, make_red(c), c->st, gate);
      launch_k(c, gemv_sym_stage2<T, NT, EpiH>, c->sym_s2_grid, NT, 0, c->stream, static_cast<const C*>(np + ns),
               static_cast<const C*>(hp + nh), c->n, c->sym2_H, CW2, c->sym2_strips, eh, make_red(c), c->st, gate);
      c->launches += 3;
      tev_end(c);
      CK(c, cudaGetLastError());
      return CCG_OK;
    }
    if (c->dual_rows && !c->dist) {   // general A, warp-per-row dual (gemv_dual_rows)
      const int CW = 256 * CT<T>::V;
      const int nstrips = (int)((c->n + CW - 1) / CW);
      const int nblk = (int)((c->nloc + c->dual_H - 1) / c->dual_H);
      tev_begin(c, 0);
      launch_k(c, gemv_dual_rows<T, NT>, nstrips * nblk, NT, 0, c->stream, A, c->lda, pfull, qloc, c->nloc, c->n,
               c->dual_H, nstrips, np, hp, gate);
      launch_k(c, part_sum_stage2<T, NT, EpiA>, c->sym_s2_grid, NT, 0, c->stream, static_cast<const C*>(np), nstrips,
               c->nloc, c->nloc, ea, make_red(c), c->st, gate);
      launch_k(c, part_sum_stage2<T, NT, EpiH>, c->sym_s2_grid, NT, 0, c->stream, static_cast<const C*>(hp), nblk, c->n,
               c->n, eh, make_red(c), c->st, gate);
      c->launches += 3;
      tev_end(c);
      CK(c, cudaGetLastError());
      return CCG_OK;
    }
    tev_begin(c, 0);
    launch_k(c, gemv_cols<T, NT, true, true, true>, dim3(c->cols_strips, c->dual_S), NT, 0, c->stream, 
        A, c->lda, pfull, qloc, c->nloc, c->n, np, hp, gate, 0);   // no L2 pinning: measured slower
    c->launches++;
    CK(c, cudaGetLastError());
    launch_k(c, gemv_h_stage2<T, NT, EpiA>, c->nstage2_grid, NT, 0, c->stream, np, c->cols_strips, c->nloc, 0, c->nloc, ea,
                                                                      make_red(c), c->st, gate);
    c->launches++;
    tev_end(c);
    CK(c, cudaGetLastError());
    TRY(post<EpiA>(c, gate));
    if (!c->dist) {
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
  static int bicgstab_setup(ccg_ctx* c, bool x0);
  static int bicgstab_iter(ccg_ctx* c);

  // ---- CGNE: loc: 0 x, 1 y, 2 r ; full: 0 p
  static int cgne_setup(ccg_ctx* c, bool x0);
  static int cgne_iter(ccg_ctx* c);

  // ---- QMR: loc: 0 x, 1 y, 2 r, 3 vt, 4 wt, 5 v, 6 w, 7 q, 8 pt, 9 d, 10 s ; full: 0 p
  static int qmr_setup(ccg_ctx* c, bool x0);
  static int qmr_iter(ccg_ctx* c);

  // ---- BiCOR: loc: 0 x, 1 y, 2 rs, 3 rh, 4 p, 5 ps, 6 q, 7 qs ; full: 0 r
  static int bicor_setup(ccg_ctx* c, bool x0);
  static int bicor_iter(ccg_ctx* c);

  // ---- CORS: loc: 0 x, 1 y, 2 r0s, 3 rh, 4 e, 5 eh, 6 h, 7 hh, 8 q ; full: 0 r, 1 qh
  static int cors_setup(ccg_ctx* c, bool x0);
  static int cors_iter(ccg_ctx* c);

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
      c->cluster_size = -1;   // none fits (MIG / MPS-limited SMs): graph path instead
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
    if (c->cluster_size < 1) {
      c->cluster_ok = false;
      return CCG_FALLBACK;
    }
    cfg.gridDim = dim3(c->cluster_size);
    at[0].val.clusterDim.x = c->cluster_size;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    if (cudaLaunchKernelEx(&cfg, kern, m, cm, c->st, reinterpret_cast<const C*>(c->A), c->lda, c->n) != cudaSuccess) {
      cudaGetLastError();   // launch refused (e.g. cluster size unavailable): graph path from now on
      c->cluster_ok = false;
      return CCG_FALLBACK;
    }
    c->launches++;
    return CCG_OK;
  }

  static int cluster_run(ccg_ctx* c, int m);

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
  static int bicg_setup(ccg_ctx* c, bool x0);
  static int bicg_iter(ccg_ctx* c);

  // ---- CGS: loc: 0 x, 1 y, 2 r, 3 rt, 4 u, 5 q, 6 v ; full: 0 p, 1 u+q
  static int cgs_setup(ccg_ctx* c, bool x0);
  static int cgs_iter(ccg_ctx* c);

  // ---- COCR: loc: 0 x, 1 y, 2 Ar, 3 p, 4 Ap ; full: 0 r
  static int cocr_setup(ccg_ctx* c, bool x0);
  static int cocr_iter(ccg_ctx* c);

  // ---- CGNR: loc: 0 x, 1 y, 2 r, 3 w, 4 z ; full: 0 p
  static int cgnr_setup(ccg_ctx* c, bool x0);
  static int cgnr_iter(ccg_ctx* c);

  // ---- TFQMR: loc: 0 x, 1 y, 2 r0*, 3 w, 4 v, 5 d, 6 A·u (even), 7 A·u2 ; full: 0 u, 1 u2
  static int tfqmr_setup(ccg_ctx* c, bool x0);
  static int tfqmr_iter(ccg_ctx* c);

  // ---- GMRES(m): loc: 0 x, 1 y, 2 w ; basis V (gm_V) ; full: 0 v_j, 2 x (restart)
  static C* Vb(ccg_ctx* c) { return reinterpret_cast<C*>(c->gm_V); }
  template <int MODE>
  static int gm_pass_launch(ccg_ctx* c, C* w, const double2* coef, double2* dst, const int* gate) {
    const bool fuse = !c->dist || c->rep;
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
  static int gmres_setup(ccg_ctx* c, bool x0);
  static int gmres_iter(ccg_ctx* c);

  // ---- BiCGstab(ℓ): loc: 0 x, 1 y, 3 r̃ ; bl_buf: r̂₀..r̂_ℓ then û₀..û_ℓ (full length each)
  static C* BLR(ccg_ctx* c, int a) { return reinterpret_cast<C*>(c->bl_buf) + (size_t)a * c->n; }
  static C* BLU(ccg_ctx* c, int a) { return BLR(c, c->bl_l + 1 + a); }
  static C* BRs(ccg_ctx* c, int a) { return BLR(c, a) + c->row0; }
  static C* BUs(ccg_ctx* c, int a) { return BLU(c, a) + c->row0; }
  static int allgather_buf(ccg_ctx* c, C* buf) {
    if (!c->dist || c->rep) return CCG_OK;
    if (c->opk == OPK_CSR || c->opk == OPK_STENCIL) return halo_exchange(c, buf);
    NK(c, c->comm->allgather_inplace(buf, (size_t)c->nloc * 2, ndt(), c->stream));
    return CCG_OK;
  }
  static int bicgstabl_setup(ccg_ctx* c, bool x0);
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
  static int bicgstabl_iter(ccg_ctx* c);

  // ---- p-BiCGSTAB: loc: 0 x, 1 y, 2 r, 3 r̃, 4 p, 5 s, 6 q, 7 y, 8 v, 9 t ; full: 0 z (r₀ at setup), 1 w
  static int pbicgstab_setup(ccg_ctx* c, bool x0);
  static int pbicgstab_iter(ccg_ctx* c);

  static int setup(ccg_ctx* c, int m, bool x0);
  static int iter(ccg_ctx* c, int m);

  // true residual ‖y − A x‖²
  static int true_residual(ccg_ctx* c);

  // right Jacobi around a solve: u₀ = D·x₀ before, x = D⁻¹·u after
  static int jac_in(ccg_ctx* c);
  static int jac_out(ccg_ctx* c);

  // ccg_apply
  static int apply(ccg_ctx* c, int op, const C* xin, C* yout);
};

