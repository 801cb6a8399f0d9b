// ccg.cu — libccg.so: the C-ABI (include/ccg.h), launch-parameter selection,
// the CUDA-graph iteration loop and handle / operator / communicator setup.
// The per-method schedules are in methods_*.cu (Engine<T>, engine.cuh).
//
// Paper mapping (PAPER.md = P:<line>):  matvec / cmatvec separated from the
// iteration (P:17, P:95 [§5]) -> ccg_set_matvec_* + the kernels of
// matvec.cuh; cgmodule's epsilon_err / maxit -> ccg_solve(tol, maxit);
// ddprecision.f90 single/double switch -> ccg_dtype.
#include "engine.cuh"

#include <nccl_device.h>   // ncclGetPeerPointer (header-only device API, NCCL 2.28)

namespace {
thread_local std::string g_create_err;   // ccg_last_error(NULL): why the last create failed
}  // namespace

// every rank's base address of an NCCL symmetric-memory window
static __global__ void p2p_resolve(ncclWindow_t w, int world, char** out) {
  const int p = threadIdx.x;
  if (p < world) out[p] = static_cast<char*>(ncclGetPeerPointer(w, 0, p));
}

// P2P mirror region: [parity 0 | parity 1] × [rep_tmp n | rep_parts world·n],
// then P2P_MAX flags (CCG_OPT_P2P, p2p.cuh)
static size_t mirror_layout(ccg_ctx* c) {
  const size_t half = ((size_t)c->n * (1 + c->world) * c->esz + 255) & ~(size_t)255;
  c->mirror_half = half;
  c->mirror_flags = 2 * half;
  return (2 * half + P2P_MAX * sizeof(uint64_t) + 4095) & ~(size_t)4095;   // NCCL_WIN_REQUIRED_ALIGNMENT
}

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
    const int wbytes = (int)((size_t)c->split_W * sizeof(C));
    auto kv = gemv_n_split<T, E::NT, E::SUR, true, false, Store<T>>;
    auto ks = gemv_n_split<T, E::NT, E::SUR, false, false, Store<T>>;
    if (wbytes > 48 * 1024) {   // strips above 48 KiB (CCG_SPLIT_KB): opt-in shared memory
      cudaFuncSetAttribute(kv, cudaFuncAttributeMaxDynamicSharedMemorySize, wbytes);
      cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, wbytes);
    }
    if (c->vec_ok)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs, kv, NT, (size_t)wbytes);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs, ks, NT, (size_t)wbytes);
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
    const char* fu = getenv("CCG_SPLIT_FUSE");
    c->split_fuse = fu ? atoi(fu) != 0 : 0;   // off: cfg3 1.3 % slower (last-CTA tail), cfg2 neutral
    if (c->rb_ticket_cap < c->split_nrb) {
      if (c->rb_ticket) cudaFree(c->rb_ticket);
      c->rb_ticket = nullptr;
      c->rb_ticket_cap = 0;
      CK(c, cudaMalloc(&c->rb_ticket, sizeof(unsigned) * c->split_nrb));
      CK(c, cudaMemsetAsync(c->rb_ticket, 0, sizeof(unsigned) * c->split_nrb, c->stream));
      c->rb_ticket_cap = c->split_nrb;
    }
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
  // QMR/BiCG dual product in the warp-per-row layout (gemv_dual_rows; one rank)
  size_t need_dual_h = 0;
  {
    const char* dr = getenv("CCG_DUAL_ROWS");
    // default on: config 3 QMR 687 -> 725 it/s, BiCG 663 -> 725; config 2 QMR
    // 86.0 -> 83.9 us/it (CCG_DUAL_ROWS=0: the column-owner dual)
    c->dual_rows = c->opk == OPK_DENSE && c->cols_ok && !c->dist && (dr ? atoi(dr) != 0 : true);
    if (c->dual_rows) {
      int occd2 = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occd2, gemv_dual_rows<T, E::NT>, NT, 0);
      const int64_t CW = (int64_t)256 * CT<T>::V;
      const int64_t nstr = (c->n + CW - 1) / CW;
      int64_t H = SYM_HMAX;
      while (H > 32 && nstr * ((c->nloc + H - 1) / H) < 2 * (int64_t)c->sm_count * std::max(1, occd2)) H /= 2;
      c->dual_H = (int)H;
      need_dual_h = (size_t)((c->nloc + H - 1) / H) * c->n * sizeof(C);
      // part_sum_stage2: one CTA per 32 outputs, at most 8 CTAs per SM
      c->sym_s2_grid = std::max(c->sym_s2_grid,
                                (int)std::max<int64_t>(1, std::min<int64_t>((c->n + 31) / 32, (int64_t)c->sm_count * 8)));
    }
  }
  size_t need_sym_h = 0;
  if (c->opk == OPK_DENSE && c->sym_ok) {
    // upper-triangle tiles: strips of CW columns × row blocks of H rows; the
    // largest H (≤ SYM_HMAX) that still fills one wave to 90 % (CCG_SYM_H;
    // config 2 BiCGSTAB at H = 32 / 64 / 128 / 256: 92.9 / 82.7 / 79.6 / 97.7
    // µs/it — longer tiles amortise the per-tile x staging and column-sum
    // reduction and leave fewer partials for stage 2).
    // Single products: CW = 256·V (gemv_sym); the dual product: 128·V.
    auto plan = [&](int64_t CW, int occ, int& strips, int& Hout, int& ntl, int2*& dtiles) -> int64_t {
      strips = (int)((c->n + CW - 1) / CW);
      auto ntiles = [&](int64_t H) {
        int64_t t = 0;
        for (int64_t cc = 0; cc < strips; ++cc) t += (std::min((cc + 1) * CW, c->n) + H - 1) / H;
        return t;
      };
      const char* he = getenv("CCG_SYM_H");
      int64_t H = he ? atoi(he) : SYM_HMAX;
      if (!he)
        while (H > 32 && 10 * ntiles(H) < 9 * (int64_t)c->sm_count * std::max(1, occ)) H /= 2;
      H = std::max<int64_t>(8, std::min<int64_t>(SYM_HMAX, (H / 8) * 8));
      Hout = (int)H;
      std::vector<int2> tl;
      const int64_t nblk = (c->n + H - 1) / H;
      for (int64_t I = 0; I < nblk; ++I)        // row-block major: concurrent CTAs read whole rows
        for (int64_t cc = 0; cc < strips; ++cc)
          if (I * H < std::min((cc + 1) * CW, c->n)) tl.push_back(make_int2((int)cc, (int)I));
      ntl = (int)tl.size();
      if (dtiles) cudaFree(dtiles);
      dtiles = nullptr;
      if (cudaMalloc(&dtiles, tl.size() * sizeof(int2)) != cudaSuccess) return -1;
      if (cudaMemcpyAsync(dtiles, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, c->stream) !=
          cudaSuccess)
        return -1;
      return nblk;
    };
    int occ1 = 0, occ2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, gemv_sym<T, E::NT, false>, NT, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, gemv_sym_dual<T, E::NT>, NT, 0);
    const int64_t nblk1 = plan((int64_t)256 * CT<T>::V, occ1, c->sym_strips, c->sym_H, c->sym_ntiles, c->sym_tiles);
    const int64_t nblk2 = plan((int64_t)128 * CT<T>::V, occ2, c->sym2_strips, c->sym2_H, c->sym2_ntiles,
                               c->sym2_tiles);
    if (nblk1 < 0 || nblk2 < 0) FAIL(c, CCG_E_CUDA, "symmetric tile tables");
    CK(c, cudaStreamSynchronize(c->stream));
    // stage 2: one CTA per 32 outputs, at most 8 CTAs per SM
    c->sym_s2_grid = (int)std::max<int64_t>(1, std::min<int64_t>((c->n + 31) / 32, (int64_t)c->sm_count * 8));
    // npart: [strips][n] (single) or 2 × [strips2][n] (dual); hpart likewise
    const size_t need = std::max((size_t)c->sym_strips, 2 * (size_t)c->sym2_strips) * c->n * sizeof(C);
    if (need > c->npart_bytes) {
      if (c->npart) cudaFree(c->npart);
      c->npart = nullptr;
      CK(c, cudaMalloc(&c->npart, need));
      c->npart_bytes = need;
    }
    need_sym_h = std::max((size_t)nblk1, 2 * (size_t)nblk2) * c->n * sizeof(C);
  }
  // workspace sized for the chosen grids
  size_t need_hpart = std::max({(size_t)std::max(c->ah_S, c->cols_ok ? c->dual_S : 1) * (size_t)c->n * sizeof(C),
                                need_sym_h, need_dual_h});
  if (c->opk == OPK_DENSE && need_hpart > c->hpart_bytes) {
    if (c->hpart) cudaFree(c->hpart);
    c->hpart = nullptr;
    CK(c, cudaMalloc(&c->hpart, need_hpart));
    c->hpart_bytes = need_hpart;
  }
  int64_t maxgrid = std::max<int64_t>({(int64_t)c->gemv_grid, (int64_t)c->ah_strips * c->ah_S,
                                       (int64_t)c->stage2_grid, (int64_t)c->pass_grid, (int64_t)c->spmv_grid,
                                       (int64_t)c->split_strips * c->split_nrb, (int64_t)c->nstage2_grid,
                                       (int64_t)c->sym_s2_grid,
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
    const int64_t calls0 = c->comm ? c->comm->calls : 0;
    CK(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int rc = E::iter(c, m);
    cudaError_t e2 = cudaStreamEndCapture(c->stream, &graph);
    c->coll_per_iter[m] = (c->comm ? c->comm->calls : 0) - calls0;
    c->stat_capture_calls += c->coll_per_iter[m];
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
      c->stat_replays++;
      c->stat_graph_coll += c->coll_per_iter[m];
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
      chunk = c->dist ? std::min(32, 2 * chunk)
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
  TRY(h2d(c, c->fftK, kh.data(), N * sizeof(C)));
  TRY(h2d(c, c->fftTw, tw.data(), half * sizeof(C)));
  CK(c, cudaMemsetAsync(c->fftW, 0, N * sizeof(C), c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
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
  c->dist = world > 1 || (options & CCG_OPT_FORCE_COMM);
  c->rep = c->dist && (options & CCG_OPT_REPLICATED);
  c->nloc = c->rep ? n : c->mnloc;      // vectors: whole (replicated) or this rank's slice
  c->row0 = c->rep ? 0 : c->mrow0;
  c->device = device;
  {
    const char* pe = getenv("CCG_PDL");
    c->pdl = !(pe && !strcmp(pe, "0"));
    const char* clr = getenv("CCG_CL_REDUNDANT");
    c->cl_redundant = !(clr && !strcmp(clr, "0"));
    const char* bf = getenv("CCG_BS_FUSE");   // BiCGSTAB P/S folds into the dense split GEMV
    c->bs_fuse = bf ? atoi(bf) != 0 : 1;
    // the S fold on the stencil / SELL SpMV: measured slower at config 5
    // (stencil 132 -> 155 us/it, CSR 211 -> 216: the latency-bound gathers
    // take two loads per neighbour), so opt-in
    const char* br = getenv("CCG_BS_FUSE_RO");
    c->bs_fuse_ro = br ? atoi(br) != 0 : 0;
    const char* bm = getenv("CCG_BS_MERGE");
    c->bs_merge = bm ? atoi(bm) != 0 : 0;
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
  CKC(cudaMemsetAsync(c->ticket, 0, sizeof(unsigned), c->stream));
  CKC(cudaMalloc(&c->rank_sum, 16 * sizeof(double2)));
  CKC(cudaMalloc(&c->all_sums, (size_t)16 * world * sizeof(double2)));
  CKC(cudaMalloc(&c->zero_gate, sizeof(int)));
  CKC(cudaMemsetAsync(c->zero_gate, 0, sizeof(int), c->stream));
  for (int i = 0; i < NLOCAL; ++i) {
    CKC(cudaMalloc(&c->loc[i], (size_t)c->nloc * c->esz));
    CKC(cudaMemsetAsync(c->loc[i], 0, (size_t)c->nloc * c->esz, c->stream));
  }
  for (int i = 0; i < NFULL; ++i) {
    CKC(cudaMalloc(&c->full[i], (size_t)n * c->esz));
    CKC(cudaMemsetAsync(c->full[i], 0, (size_t)n * c->esz, c->stream));
  }
  if (c->rep) {
    CKC(cudaMalloc(&c->rep_tmp, (size_t)n * c->esz));
    CKC(cudaMalloc(&c->rep_parts, (size_t)n * world * c->esz));
  }
  if ((options & CCG_OPT_P2P) && !(c->rep && world <= P2P_MAX)) {
    c->err = "CCG_OPT_P2P needs CCG_OPT_REPLICATED, a communicator (world > 1 or CCG_OPT_FORCE_COMM) and world <= 8";
    return bail(CCG_E_ARG);
  }
  c->p2p = (options & CCG_OPT_P2P) != 0;
  if (c->dist) {
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
      uint8_t own_id[128];
      if (!nccl_id) {   // world == 1 with CCG_OPT_FORCE_COMM: a one-rank communicator
        if (ccg_get_unique_id(own_id) != CCG_OK) { c->err = g_create_err; return bail(CCG_E_NCCL); }
        nccl_id = own_id;
      }
      int rc = nc->init(world, rank, nccl_id);
      if (rc) { c->err = nc->err; return bail(CCG_E_NCCL); }
      if (c->p2p) {   // symmetric-memory window + every rank's address of it
        c->mirror_bytes = mirror_layout(c);
        rc = nc->window_alloc(c->mirror_bytes, &c->mirror, &c->win);
        if (rc) { c->err = nc->err; return bail(rc == -3 ? CCG_E_CAPABILITY : CCG_E_NCCL); }
        char** dptr = nullptr;
        CKC(cudaMalloc(&dptr, sizeof(char*) * P2P_MAX));
        p2p_resolve<<<1, 32, 0, c->stream>>>(c->win, world, dptr);
        cudaError_t e1 = cudaGetLastError();
        if (e1 == cudaSuccess)
          e1 = cudaMemcpyAsync(c->peer_base, dptr, sizeof(char*) * world, cudaMemcpyDeviceToHost, c->stream);
        if (e1 == cudaSuccess) e1 = cudaStreamSynchronize(c->stream);
        cudaFree(dptr);
        CKC(e1);
      }
    }
    if (c->p2p) {
      if (lg) {   // loopback: the peers' regions are filled in by the group
        c->mirror_bytes = mirror_layout(c);
        CKC(cudaMalloc(&c->mirror, c->mirror_bytes));
        c->peer_base[rank] = static_cast<char*>(c->mirror);
      }
      CKC(cudaMemsetAsync(c->mirror, 0, c->mirror_bytes, c->stream));
      CKC(cudaMalloc(&c->p2p_ctr, 2 * sizeof(uint64_t)));
      CKC(cudaMemsetAsync(c->p2p_ctr, 0, 2 * sizeof(uint64_t), c->stream));
      CKC(cudaStreamSynchronize(c->stream));
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
  } else if (options & CCG_OPT_P2P) {   // every rank sees every rank's mirror region
    for (int r = 0; r < world; ++r)
      for (int p = 0; p < world; ++p) hs[r]->peer_base[p] = static_cast<char*>(hs[p]->mirror);
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
    // complex-symmetric A, one rank: products from the upper triangle only
    // (matvec.cuh gemv_sym; CCG_SYMV=0 reads all of A).  Declared by the caller
    // (CCG_FLAG_SYMMETRIC) or detected exactly here: A = Aᵀ bit for bit, one
    // read of A when it holds, a few tiles when it does not (CCG_SYM_DETECT=0
    // skips the test).  The matrix is borrowed unmodified until the next
    // set_matvec (ccg.h), so the property holds for every product.
    const char* sv = getenv("CCG_SYMV");
    const char* sd = getenv("CCG_SYM_DETECT");
    const bool usable = !c->dist && c->vec_ok && (c->n % (c->esz == 8 ? 2 : 1)) == 0 && !(sv && !strcmp(sv, "0"));
    c->sym_state = 0;
    if (usable && (flags & CCG_FLAG_SYMMETRIC)) {
      c->sym_state = 1;
    } else if (usable && !(sd && !strcmp(sd, "0"))) {
      int* bad = nullptr;
      CK(c, cudaMalloc(&bad, sizeof(int)));
      CK(c, cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
      const int grid = c->sm_count * 8;
      if (c->dtype == CCG_C64)
        sym_check<float><<<grid, 256, 0, c->stream>>>(static_cast<const float2*>(A_local), lda, c->n, bad);
      else
        sym_check<double><<<grid, 256, 0, c->stream>>>(static_cast<const double2*>(A_local), lda, c->n, bad);
      int hbad = 1;
      const cudaError_t e1 = cudaGetLastError();
      const cudaError_t e2 = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
      const cudaError_t e3 = cudaStreamSynchronize(c->stream);
      cudaFree(bad);
      CK(c, e1);
      CK(c, e2);
      CK(c, e3);
      if (!hbad) c->sym_state = 2;
    }
    c->sym_ok = c->sym_state != 0;
  }
  {
    // L2-resident rows (matvec.cuh): ~80 MB of A kept in the
    // 126 MB L2 between the products of a solve; 0 when A is >> L2
    const char* pe = getenv("CCG_L2_PIN_MB");
    const double pin_bytes = (pe ? atof(pe) : 80.0) * 1e6;
    const double abytes = (double)nloc * (double)c->n * (double)c->esz * (c->sym_ok ? 0.5 : 1.0);
    c->l2_pin = pin_bytes <= 0 || abytes < 32e6 ? 0      // small A stays in L2 without help
                : abytes <= pin_bytes ? 64 : (int)floor(64.0 * pin_bytes / abytes);
  }
  {
    // small L2-resident systems: the whole loop in one cluster (cluster.cuh)
    const char* ce = getenv("CCG_CLUSTER");
    const char* cb = getenv("CCG_CLUSTER_MAXBYTES");
    const double maxb = cb ? atof(cb) : 4.0 * 1024 * 1024;
    c->cluster_ok = !c->dist && !(ce && !strcmp(ce, "0")) &&
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
  // validate structure and compute the halo width on the host (one-time copy).
  // A local failure is recorded, not returned: with several ranks every rank
  // first enters the halo-width allgather, so an input error on one rank is an
  // error on all of them instead of a hang in the collective.
  int lcode = CCG_OK;
  std::string lmsg;
  auto lfail = [&](int code, const char* m) {
    if (lcode == CCG_OK) { lcode = code; lmsg = m; }
  };
  std::vector<int32_t> rp(nloc + 1), ci(nnz_local);
  int64_t halo = 0;
  CK(c, cudaMemcpy(rp.data(), rowptr, (nloc + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (nnz_local) CK(c, cudaMemcpy(ci.data(), colind, nnz_local * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (rp[0] != 0 || rp[nloc] != nnz_local) lfail(CCG_E_DIM, "rowptr[0] != 0 or rowptr[nloc] != nnz");
  for (int64_t i = 0; i < nloc && lcode == CCG_OK; ++i) {
    if (rp[i + 1] < rp[i]) { lfail(CCG_E_ARG, "rowptr not nondecreasing"); break; }
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t j = ci[k];
      if (j < 0 || j >= c->n) { lfail(CCG_E_ARG, "column index out of range"); break; }
      if (j < row0) halo = std::max<int64_t>(halo, row0 - j);
      if (j >= row0 + nloc) halo = std::max<int64_t>(halo, j - (row0 + nloc) + 1);
    }
  }
  if (lcode == CCG_OK && c->dist && !c->rep && halo > nloc)
    lfail(CCG_E_ARG, "CSR columns reach beyond the neighbour ranks (halo > nloc)");
  if (c->dist && !c->rep) {
    // all ranks use the same (maximum) halo width so that sends match receives,
    // and share their validation status
    const int64_t mine[2] = {halo, (int64_t)lcode};
    int64_t* dh = nullptr;
    CK(c, cudaMalloc(&dh, sizeof(int64_t) * 2 * c->world));
    CK(c, cudaMemcpyAsync(dh + 2 * c->rank, mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream));
    int r = c->comm->allgather(dh + 2 * c->rank, dh, 2, CT_I64, c->stream);
    if (r) { cudaFree(dh); FAIL(c, r, c->comm->err); }
    std::vector<int64_t> hs(2 * c->world);
    CK(c, cudaMemcpyAsync(hs.data(), dh, sizeof(int64_t) * 2 * c->world, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    cudaFree(dh);
    if (lcode != CCG_OK) FAIL(c, lcode, lmsg);
    for (int p = 0; p < c->world; ++p) {
      if (hs[2 * p + 1] != CCG_OK)
        FAIL(c, (int)hs[2 * p + 1], "ccg_set_matvec_csr failed on rank " + std::to_string(p));
      halo = std::max(halo, hs[2 * p]);
    }
    if (halo > nloc) FAIL(c, CCG_E_ARG, "halo > nloc on some rank");
  } else if (lcode != CCG_OK) {
    FAIL(c, lcode, lmsg);
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
      TRY(h2d(c, c->sell_off, off.data(), nsl * sizeof(int64_t)));
      TRY(h2d(c, c->sell_width, wid.data(), nsl * sizeof(int32_t)));
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
    TRY(h2d(c, c->csr_blocks, bl.data(), bl.size() * sizeof(int32_t)));
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
  // launch bound "4 CTAs/SM" (≤ 64 registers, 32 warps/SM): the stencil is
  // latency-bound; interleaved A/B at config 5 (ab/cfg5_stencil_minb.jsonl):
  // BiCGSTAB 142.9 -> 129.8 us/it, CORS 174.3 -> 155.8, COCR 101.5 -> 93.4
  const char* smb = getenv("CCG_STENCIL_MINB");
  c->stencil_minb = smb && atoi(smb) == 1 ? 1 : smb && atoi(smb) == 3 ? 3 : 4;
  const char* sro = getenv("CCG_STENCIL_REALO");
  c->stencil_realo = !(sro && atoi(sro) == 0);
  if (zc) {
    c->szc = std::max(1, atoi(zc));
  } else {
    // the longest z-march of 16, 8, 4 planes that still gives ≥ 3 CTAs per SM (fewer z-chunk halo planes
    // re-read, fewer reduction slots; with the loop unrolled by 2 — ab/cfg5_stencil_zc_unroll2.jsonl —
    // 16 beats 8 at 128³: BiCGSTAB 121.0 → 119.3 µs/it, CORS 149.4 → 144.6, CGS 117.8 → 112.1)
    const int64_t tiles = ((nx + 31) / 32) * ((ny + 7) / 8);
    c->szc = 4;
    for (int z : {16, 8}) {
      if (tiles * ((c->snzl + z - 1) / z) >= 3 * (int64_t)c->sm_count) { c->szc = z; break; }
    }
  }
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
  {
    // passes 2-4 fused (one kx plane per CTA), opt-in (CCG_FFT_YZ=1) where a
    // plane fits in shared memory: measured neutral at config 4 (BiCGSTAB
    // 79.7 vs 79.6 µs/it; the fused kernel takes 20 µs on 128 CTAs — one
    // 16-warp CTA per SM cannot hide the per-stage latency the separate
    // passes hide with 2+ CTAs per SM)
    const char* fy = getenv("CCG_FFT_YZ");
    const size_t smp = (size_t)g.Y2 * (g.Z2 + 1) * (c->dtype == CCG_C64 ? 8 : 16);
    c->fft_yz = smp <= 200 * 1024 && fy && atoi(fy) != 0;
  }
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
  // a bad entry is recorded, not returned, so that with several ranks every
  // rank still enters the allgathers below (no hang); the status is agreed
  int lcode = CCG_OK;
  for (int64_t i = 0; i < c->mnloc; ++i) {
    double re, im;
    if (es == 8) { re = reinterpret_cast<float*>(hd.data())[2 * i]; im = reinterpret_cast<float*>(hd.data())[2 * i + 1]; }
    else { re = reinterpret_cast<double*>(hd.data())[2 * i]; im = reinterpret_cast<double*>(hd.data())[2 * i + 1]; }
    if (!(std::isfinite(re) && std::isfinite(im)) || (re == 0.0 && im == 0.0)) { lcode = CCG_E_ARG; break; }
    const std::complex<double> inv = 1.0 / std::complex<double>(re, im);
    if (es == 8) {
      reinterpret_cast<float*>(hinv.data())[2 * i] = (float)inv.real();
      reinterpret_cast<float*>(hinv.data())[2 * i + 1] = (float)inv.imag();
    } else {
      reinterpret_cast<double*>(hinv.data())[2 * i] = inv.real();
      reinterpret_cast<double*>(hinv.data())[2 * i + 1] = inv.imag();
    }
  }
  if (c->dist) {
    int64_t* dcode = nullptr;
    const int64_t mine = lcode;
    std::vector<int64_t> all(c->world);
    CK(c, cudaMalloc(&dcode, sizeof(int64_t) * c->world));
    CK(c, cudaMemcpyAsync(dcode + c->rank, &mine, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    int r = c->comm->allgather(dcode + c->rank, dcode, 1, CT_I64, c->stream);
    if (!r) {
      cudaMemcpyAsync(all.data(), dcode, sizeof(int64_t) * c->world, cudaMemcpyDeviceToHost, c->stream);
      cudaStreamSynchronize(c->stream);
    }
    cudaFree(dcode);
    if (r) FAIL(c, r, c->comm->err);
    for (auto v : all) if (v != CCG_OK) lcode = (int)v;
  }
  if (lcode != CCG_OK) FAIL(c, lcode, "Jacobi: diagonal entries must be finite and nonzero (on every rank)");
  const size_t full = (size_t)c->n * es;
  if (!c->jac_d) CK(c, cudaMalloc(&c->jac_d, full));
  if (!c->jac_dinv) CK(c, cudaMalloc(&c->jac_dinv, full));
  if (!c->jac_tmp) CK(c, cudaMalloc(&c->jac_tmp, full));
  TRY(h2d(c, static_cast<char*>(c->jac_d) + (size_t)c->mrow0 * es, hd.data(), hd.size()));
  TRY(h2d(c, static_cast<char*>(c->jac_dinv) + (size_t)c->mrow0 * es, hinv.data(), hinv.size()));
  if (c->dist) {
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
    CK(c, cudaMemsetAsync(c->bl_buf, 0, need, c->stream));
    c->bl_bytes = need;
  }
  invalidate_graphs(c);   // buffer layout depends on ℓ
  if (!c->gm_dev) {
    CK(c, cudaMalloc(&c->gm_dev, sizeof(GmDev)));
    CK(c, cudaMemsetAsync(c->gm_dev, 0, sizeof(GmDev), c->stream));
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
    CK(c, cudaMemsetAsync(c->gm_dev, 0, sizeof(GmDev), c->stream));
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
    CK(c, cudaMemsetAsync(c->gm_ticket, 0, sizeof(unsigned), c->stream));
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
  if (c->opk == OPK_CSR && op != CCG_OP_A && (!(c->flags & CCG_FLAG_SYMMETRIC) || (c->dist && !c->rep)))
    FAIL(c, CCG_E_CAPABILITY, "CSR Aᴴ/Aᵀ needs CCG_FLAG_SYMMETRIC and world == 1 (or replicated vectors)");
  if (c->opk == OPK_CALLBACK && !(c->cb_caps & (op == CCG_OP_A ? CCG_CB_A : op == CCG_OP_AH ? CCG_CB_AH : CCG_CB_AT)))
    FAIL(c, CCG_E_CAPABILITY, "the user callback does not provide this product");
  CK(c, cudaSetDevice(c->device));
  struct PinGuard {
    ccg_ctx* c;
    ~PinGuard() { c->pin_on = false; }
  } pin_guard{c};
  c->pin_on = c->opk == OPK_DENSE && c->l2_pin > 0;
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
  if (needs_ah(method) && c->opk == OPK_CSR && (!(c->flags & CCG_FLAG_SYMMETRIC) || (c->dist && !c->rep)))
    FAIL(c, CCG_E_CAPABILITY, "method needs Aᴴ; CSR provides it only with CCG_FLAG_SYMMETRIC and world == 1");
  if (c->opk == OPK_CALLBACK && (!(c->cb_caps & CCG_CB_A) || (needs_ah(method) && !(c->cb_caps & CCG_CB_AH))))
    FAIL(c, CCG_E_CAPABILITY, "the user callback does not provide the products this method needs");
  CK(c, cudaSetDevice(c->device));
  struct PinGuard {
    ccg_ctx* c;
    ~PinGuard() { c->pin_on = false; }
  } pin_guard{c};
  c->pin_on = c->opk == OPK_DENSE && c->l2_pin > 0;
  c->launches = 0;
  c->ms_a = c->ms_ah = 0;
  c->n_a = c->n_ah = 0;
  c->stat_replays = c->stat_graph_coll = c->stat_capture_calls = 0;
  const int64_t calls_start = c->comm ? c->comm->calls : 0;
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
  if (c->opk == OPK_DENSE && c->cluster_ok && !c->dist && !c->timing && method != CCG_GMRES &&
      method != CCG_BICGSTABL && !c->jac_dinv) {
    // small dense system: setup, every iteration and the true residual in ONE
    // cluster launch (cluster.cuh); maxit and the stopping rule live in the State
    c->cl_method = method;
    c->cl_has_x0 = has_x0 ? 1 : 0;
    rc = c->dtype == CCG_C64 ? Engine<float>::cluster_run(c, method) : Engine<double>::cluster_run(c, method);
    if (rc && rc != CCG_FALLBACK) return rc;
  }
  if (!(c->opk == OPK_DENSE && c->cluster_ok && !c->dist && !c->timing && method != CCG_GMRES &&
        method != CCG_BICGSTABL && !c->jac_dinv)) {
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
  if (c->pin_on) {   // the pinned rows of A back to normal L2 priority
    const int g = c->sm_count * 8;
    if (c->dtype == CCG_C64)
      l2_demote<float><<<g, 256, 0, c->stream>>>(reinterpret_cast<const float2*>(c->A), c->lda, c->mnloc, c->n, c->l2_pin);
    else
      l2_demote<double><<<g, 256, 0, c->stream>>>(reinterpret_cast<const double2*>(c->A), c->lda, c->mnloc, c->n,
                                                  c->l2_pin);
    CK(c, cudaGetLastError());
    c->launches++;
    c->pin_on = false;
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
  c->stat_eager_coll = (c->comm ? c->comm->calls : 0) - calls_start - c->stat_capture_calls;
  res->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  return CCG_OK;
}

int ccg_get_history(ccg_handle c, double* rel_res, int32_t cap, int32_t* len) {
  if (!c || !len) return CCG_E_ARG;
  if (!c->hist || c->hist_len == 0) { *len = 0; return CCG_OK; }
  int32_t m = std::min<int32_t>(cap, c->hist_len);
  if (m > 0 && rel_res) {   // ordered after the solve's kernels on the (non-blocking) library stream
    CK(c, cudaMemcpyAsync(rel_res, c->hist, sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
  }
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

int ccg_get_stat(ccg_handle c, int32_t key, int64_t* value) {
  if (!c || !value) return CCG_E_ARG;
  switch (key) {
    case CCG_STAT_COMM_KIND: *value = c->comm ? c->comm->kind : 0; break;
    case CCG_STAT_GRAPH_REPLAYS: *value = c->stat_replays; break;
    case CCG_STAT_GRAPH_COLLECTIVES: *value = c->stat_graph_coll; break;
    case CCG_STAT_EAGER_COLLECTIVES: *value = c->stat_eager_coll; break;
    case CCG_STAT_WORLD: *value = c->world; break;
    case CCG_STAT_REPLICATED: *value = c->rep ? 1 : 0; break;
    case CCG_STAT_P2P_EXCHANGES: *value = c->p2p_calls; break;
    case CCG_STAT_SYMMETRIC: *value = c->opk == OPK_DENSE ? c->sym_state : 0; break;
    default: FAIL(c, CCG_E_ARG, "unknown stat key");
  }
  return CCG_OK;
}

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
  if (c->mirror) {
    NcclComm* nc = c->win ? dynamic_cast<NcclComm*>(c->comm) : nullptr;
    if (nc) nc->window_free(c->mirror, c->win);
    else cudaFree(c->mirror);
    c->mirror = nullptr;
  }
  if (c->p2p_ctr) cudaFree(c->p2p_ctr);
  if (c->rb_ticket) cudaFree(c->rb_ticket);
  delete c->comm;
  c->comm = nullptr;
  for (int i = 0; i < NLOCAL; ++i) if (c->loc[i]) cudaFree(c->loc[i]);
  for (int i = 0; i < NFULL; ++i) if (c->full[i]) cudaFree(c->full[i]);
  if (c->wfull) cudaFree(c->wfull);
  if (c->rep_tmp) cudaFree(c->rep_tmp);
  if (c->rep_parts) cudaFree(c->rep_parts);
  if (c->hpart) cudaFree(c->hpart);
  if (c->npart) cudaFree(c->npart);
  if (c->sym_tiles) cudaFree(c->sym_tiles);
  if (c->sym2_tiles) cudaFree(c->sym2_tiles);
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
