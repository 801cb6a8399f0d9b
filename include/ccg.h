/*
 * ccg.h — C-ABI of libccg.so, the B200 (sm_100a) hot path of the complex
 * conjugate-gradient family catalogued by CCGPAK (Flatau, arXiv:1208.4869).
 *
 * Citations: "P:<n>" = /root/reference/PAPER.md line n (its section in
 * brackets); "S:<n>" = SPEC.md line n; "SURVEY §x" = /root/repo/SURVEY.md.
 *
 * The paper's contract is a user-supplied matrix-vector product kept apart
 * from the Krylov iteration (P:17 [abstract]: "mechanism for matrix times
 * vector multiplication which is separated from the conjugate gradient
 * iterations itself"; P:95 [§5]: matvec / cmatvec in module arraymodule), a
 * configuration record carrying the tolerance epsilon_err and maxit (P:95
 * [§5], module cgmodule), and a single/double precision switch (P:17, P:95
 * [§5], ddprecision.f90).  This header maps them to:
 *
 *   ccg_create             precision switch (CCG_C64 / CCG_C128) + device/comm
 *   ccg_set_matvec_dense   matvec/cmatvec over a dense row-major matrix
 *   ccg_set_matvec_csr     matvec over a CSR matrix ("own sparse matrix scheme")
 *   ccg_apply              one product A·x, Aᴴ·x or Aᵀ·x (per-matvec parity hook)
 *   ccg_solve              one solve by BiCGSTAB / CGNE / QMR (P:57 [§2.1]) or
 *                          BiCOR / CORS (P:69 [§2.4]) with epsilon_err, maxit
 *   ccg_destroy
 *
 * Conventions for every function:
 *  - Complex numbers are interleaved (re, im) pairs: CCG_C64 = 2 x float
 *    (8 bytes), CCG_C128 = 2 x double (16 bytes).  Vectors are contiguous.
 *  - Return value: a ccg_err (0 = CCG_OK).  On error nothing is half-done
 *    that the caller must undo; ccg_last_error(h) gives a one-line reason.
 *    Solver OUTCOMES (max iterations, breakdown, ...) are not errors: they
 *    are reported in ccg_result.status.
 *  - Multi-GPU: one process per GPU (world ranks).  Every rank calls
 *    ccg_apply / ccg_solve collectively with the same arguments except the
 *    vector pointers, which hold that rank's row slice; every rank receives
 *    the same ccg_result.
 *  - No CPU fallback: every arithmetic step runs in libccg's CUDA kernels.
 *    Without a usable CUDA device ccg_create returns CCG_E_CUDA.
 */
#ifndef CCG_H_
#define CCG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ccg_ctx* ccg_handle;

/* Working precision ("simple to switch between single and double
 * precisions"; ddprecision.f90).  Matrix, vectors and matvec
 * arithmetic are in this precision; reductions (dot products, norms) are
 * accumulated in fp64 and the recurrence scalars are kept in fp64. */
typedef enum { CCG_C64 = 0, CCG_C128 = 1 } ccg_dtype;

/* Methods on the hot path (BASELINE.json north_star).  BiCGSTAB, CGNE, QMR:
 * PIM90 set (P:57 [§2.1]; QMR as corrected, P:101 [§6]).  BiCOR, CORS:
 * Carpentieri-Jing-Huang (P:69 [§2.4]).  Recurrences: SURVEY §8(c) O1-O5 /
 * DESIGN.md.  The rest of the catalogue on the same kernels (SURVEY §8(f)
 * NEXT-3): BiCG ("bigcg"), CGS, CGNR ("cgmr", read as CGNR) of the PIM90 set
 * (P:57 [§2.1]) and COCR (P:87 [§3.4]; meant for complex-symmetric A = Aᵀ —
 * the library does not check symmetry).  Recurrences: DESIGN.md §2.
 * TFQMR (P:57 [§2.1], "QMR and TFQMR ... changed") is the transpose-free QMR
 * smoothing of CGS.  Operator needs: BiCGSTAB, CORS, CGS, COCR, TFQMR -> A·x
 * only; CGNE, QMR, BiCOR, BiCG, CGNR -> A·x and Aᴴ·x. */
typedef enum {
  CCG_BICGSTAB = 0,
  CCG_CGNE = 1,
  CCG_QMR = 2,
  CCG_BICOR = 3,
  CCG_CORS = 4,
  CCG_BICG = 5,
  CCG_CGS = 6,
  CCG_COCR = 7,
  CCG_CGNR = 8,
  CCG_TFQMR = 9,  /* P:57 [§2.1]; stops on Freund's bound τ_m·√(m+1) ≤ tol·‖r₀‖ (R9) */
  CCG_GMRES = 10, /* restarted GMRES(m), P:57 [§2.1] "rgmres"; m from ccg_set_gmres_restart (default 30);
                     iterations = Arnoldi steps, + one A·x per restart (R12-R15) */
  CCG_BICGSTABL = 11, /* BiCGstab(ℓ), P:79 [§3.1] (vanilla); ℓ from ccg_set_bicgstab_ell (default 2);
                        iterations = BiCG steps, two A·x each (R16-R18) */
  CCG_PBICGSTAB = 12 /* pipelined BiCGSTAB (SURVEY §8(f) NEXT-2 iii): BiCGSTAB's iterates in exact
                        arithmetic with two reduction phases per iteration, each independent of the
                        product that follows it (2 A·x per iteration + 2 at setup, the last skipped) */
} ccg_method;

/* The three products of the operator module: A·x (matvec),
 * Aᴴ·x (cmatvec, conjugate transpose), Aᵀ·x (unconjugated transpose). */
typedef enum { CCG_OP_A = 0, CCG_OP_AH = 1, CCG_OP_AT = 2 } ccg_op;

/* Flags for ccg_set_matvec_*.  CCG_FLAG_SYMMETRIC: caller asserts A == Aᵀ
 * (complex symmetric, unconjugated; the DDA matrices of P:47 §1
 * and the COCG/COCR family of P:69 §2.4, §3.4).  Not verified by the
 * library.  For CSR it enables Aᴴ·x = conj(A·conj(x)) (single GPU only); for
 * a dense matrix on one rank the products read only the upper triangle
 * j ≥ i (half of A's bytes; the strictly-lower triangle is never read). */
enum { CCG_FLAG_SYMMETRIC = 1 };

typedef enum {
  CCG_OK = 0,
  CCG_E_ARG = -1,        /* NULL handle/pointer, bad enum, tol < 0, maxit < 1, misaligned */
  CCG_E_DIM = -2,        /* sizes inconsistent with the handle (n, nloc, row0, lda, nnz) */
  CCG_E_CAPABILITY = -3, /* method/op needs Aᴴ (or Aᵀ) the operator cannot provide */
  CCG_E_STATE = -4,      /* ccg_apply/ccg_solve before any ccg_set_matvec_* */
  CCG_E_CUDA = -5,       /* CUDA runtime error (text in ccg_last_error) */
  CCG_E_NCCL = -6,       /* NCCL error or NCCL unavailable with world > 1 */
  CCG_E_OOM = -7,        /* device allocation failed */
  CCG_E_USER = -8        /* a user matvec callback returned non-zero */
} ccg_err;

/* Solve outcome (mirrors SPEC SolverOutcome). */
typedef enum {
  CCG_CONVERGED = 0,         /* ‖r_k‖ ≤ tol·‖r_0‖ on the recurrence residual */
  CCG_MAXIT = 1,             /* maxit outer iterations without convergence */
  CCG_BREAKDOWN = 2,         /* a recurrence divisor was exactly 0 (breakdown_code names it) */
  CCG_FALSE_CONVERGENCE = 3, /* converged on the recurrence but true residual > 10·tol */
  CCG_NONFINITE = 4          /* a NaN/Inf reached a recurrence scalar */
} ccg_status;

/* Breakdown codes: which divisor vanished (SURVEY §8(c) O1-O5 names). */
typedef enum {
  CCG_BD_NONE = 0, CCG_BD_RHO = 1, CCG_BD_SIGMA = 2, CCG_BD_TT = 3, CCG_BD_OMEGA = 4,
  CCG_BD_PI = 5, CCG_BD_DELTA = 6, CCG_BD_EPSILON = 7, CCG_BD_BETA = 8, CCG_BD_XI = 9,
  CCG_BD_VNORM = 10, CCG_BD_WNORM = 11, CCG_BD_GAMMA = 12
} ccg_breakdown;

typedef struct {
  int32_t status;         /* ccg_status */
  int32_t iterations;     /* outer iterations completed; BiCGSTAB half-step exit counts k */
  int32_t matvecs_a;      /* A·x applications by the recurrence (setup included, final check excluded) */
  int32_t matvecs_ah;     /* Aᴴ·x applications */
  int32_t breakdown_code; /* ccg_breakdown */
  int32_t half_step;      /* 1 if BiCGSTAB exited on ‖s‖ */
  double rec_rel_res;     /* last recurrence residual ‖r_k‖/‖r_0‖ */
  double true_rel_res;    /* ‖y − A·x̂‖/‖r_0‖ recomputed at exit */
  double wall_ms;         /* host wall time of the call */
} ccg_result;

/* NCCL unique id for world > 1: rank 0 calls this, the caller broadcasts the
 * 128 bytes (e.g. over a torch.distributed process group) and every rank
 * passes them to ccg_create.  Returns CCG_E_NCCL if NCCL is unavailable. */
int ccg_get_unique_id(uint8_t id[128]);

/* Create a handle for an n×n system in precision dt.
 *   world, rank : number of ranks (one GPU each) and this rank; world = 1 for a
 *                 single GPU.  With world > 1 rank r owns rows
 *                 [r·n/world, (r+1)·n/world) (n % world == 0 required, else CCG_E_DIM).
 *   nccl_id     : 128 bytes from ccg_get_unique_id (NULL iff world == 1).
 *   device      : CUDA device ordinal this handle uses.
 *   cuda_stream : cudaStream_t to order work on, or NULL for a private stream.
 * Ownership: the library owns all workspace (Krylov vectors, reduction slots,
 * NCCL communicator, CUDA graphs) and frees it in ccg_destroy. */
int ccg_create(ccg_handle* h, ccg_dtype dt, int64_t n, int world, int rank,
               const uint8_t* nccl_id, int device, void* cuda_stream);

/* ccg_create with options.  CCG_OPT_REPLICATED (world > 1; SURVEY §8(f)
 * NEXT-2 ii): every rank keeps the WHOLE Krylov vectors (n elements; vector
 * passes and dot products run redundantly and identically on every rank), the
 * operator stays row-sharded.  A product then costs one collective — the
 * allgather of its output rows (A·x), or of each rank's full-length partial,
 * summed in rank order (dense Aᴴ·x) — and no reduction phase needs any
 * collective: BiCGSTAB does 2 collectives per iteration instead of 2 input
 * allgathers + 4 scalar allgathers.  The API is unchanged: vector arguments
 * are still this rank's nloc-row slices.  Costs n·s per vector pass per rank
 * (negligible against a dense row block). */
/* CCG_OPT_FORCE_COMM: take the sharded code path (NCCL collectives, the fixed
 * chunk schedule, graph-captured collectives) even with world == 1, where a
 * one-rank NCCL communicator is created (nccl_id may then be NULL).  Every
 * collective is then an identity, so results equal the world == 1 path up to
 * summation order; it exists to run the NCCL data plane on one GPU.  Combine
 * with CCG_OPT_REPLICATED for the replicated-vector mode. */
/* CCG_OPT_P2P (with CCG_OPT_REPLICATED; world <= 8, one NVLink/NVSwitch
 * domain; SURVEY §8(f) NEXT-2 i): the gather that ends every replicated-mode
 * product (rows of A·x, dense Aᴴ partials) is fused into the product kernel's
 * epilogue — each output element is stored directly into every rank's
 * buffer through an NCCL symmetric-memory window (ncclCommWindowRegister,
 * ncclGetPeerPointer), followed by a release flag per rank and an acquire
 * wait; no NCCL collective remains on the product path.  Double-buffered by
 * a device-side exchange epoch.  CCG_E_CAPABILITY if NCCL has no windows.
 * (The user-callback operator keeps the NCCL allgather.) */
enum { CCG_OPT_REPLICATED = 1, CCG_OPT_FORCE_COMM = 2, CCG_OPT_P2P = 4 };
int ccg_create_ex(ccg_handle* h, ccg_dtype dt, int64_t n, int world, int rank,
                  const uint8_t* nccl_id, int device, void* cuda_stream, uint32_t options);

/* Validation hook for the sharded path on ONE GPU: creates `world` (≥ 2)
 * handles hs[0..world-1] for ranks 0..world-1 of an n×n system on `device`,
 * wired to an in-process loopback communicator instead of NCCL (every
 * collective becomes a host-side barrier plus device-to-device copies, so no
 * kernel waits on another rank).  Each handle must be driven by its own host
 * thread, all calling the same collective functions in the same order.  The
 * handles are otherwise identical to ccg_create(..., world, rank, ...) ones
 * (same kernels, same row ownership); each is released with ccg_destroy.
 * On error no handle is left allocated. */
int ccg_create_loopback_group(ccg_handle* hs, int world, ccg_dtype dt, int64_t n, int device);
/* Same with ccg_create_ex options (e.g. CCG_OPT_REPLICATED). */
int ccg_create_loopback_group_ex(ccg_handle* hs, int world, ccg_dtype dt, int64_t n, int device,
                                 uint32_t options);

/* Dense operator (matvec + cmatvec of a row-major matrix; P:95 [§5]).
 *   A_local : DEVICE pointer to this rank's rows, row-major, nloc × n with
 *             leading dimension lda ≥ n (elements).  Borrowed: the caller keeps
 *             it alive and unmodified until ccg_destroy or the next set_matvec.
 *   row0, nloc : must equal the handle's row range (rank·n/world, n/world).
 *   flags   : CCG_FLAG_SYMMETRIC or 0.  With the flag and world == 1 every
 *             product (A, Aᴴ, Aᵀ; QMR's A·p and Aᴴ·q in one pass) reads only
 *             the upper triangle j ≥ i: y_i = Σ_{j≥i} A_ij x_j + Σ_{j<i} A_ji x_j
 *             (same products up to summation order; env CCG_SYMV=0 reads all
 *             of A).  Without the flag (world == 1) the call tests A = Aᵀ bit
 *             for bit on the device — one read of A if it holds, a few tiles
 *             if not — and takes the same path when it holds
 *             (CCG_STAT_SYMMETRIC tells which; env CCG_SYM_DETECT=0 skips the
 *             test).  With world > 1 the flag is informational.
 * Supports CCG_OP_A, CCG_OP_AH, CCG_OP_AT. */
int ccg_set_matvec_dense(ccg_handle h, const void* A_local, int64_t row0, int64_t nloc,
                         int64_t lda, uint32_t flags);

/* CSR operator, rows [row0, row0+nloc) of the global matrix.
 *   rowptr : DEVICE int32[nloc+1], rowptr[0] == 0, nondecreasing, rowptr[nloc] == nnz_local.
 *   colind : DEVICE int32[nnz_local], GLOBAL column indices in [0, n).  With world > 1
 *            every column must lie within [row0 − h, row0 + nloc + h) for a halo
 *            width h ≤ nloc (neighbour ranks only), else CCG_E_ARG.
 *   vals   : DEVICE complex[nnz_local] in the handle's precision.
 *   Borrowed like the dense matrix.  Supports CCG_OP_A; CCG_OP_AH / CCG_OP_AT
 *   only with CCG_FLAG_SYMMETRIC and world == 1, else CCG_E_CAPABILITY. */
int ccg_set_matvec_csr(ccg_handle h, const int32_t* rowptr, const int32_t* colind,
                       const void* vals, int64_t row0, int64_t nloc, int64_t nnz_local,
                       uint32_t flags);

/* Matrix-free 7-point stencil operator on an nx × ny × nz lattice (x fastest,
 * global index i = ix + nx·(iy + ny·iz)), Dirichlet boundaries:
 *   (A u)_i = d·u_i + ox·(u_{i−1} + u_{i+1}) + oy·(u_{i−nx} + u_{i+nx}) + oz·(u_{i−nx·ny} + u_{i+nx·ny}),
 * terms whose neighbour lies outside the lattice omitted.  This is the paper's
 * "own sparse matrix scheme" hook (P:95 [§5]: matvec / cmatvec written for a
 * structured operator) for config 5's shifted Helmholtz operator (BJ:11:
 * d = 6 − k²(1 + i/2), ox = oy = oz = −1): no matrix is
 * stored, so one product moves 2·n complex values instead of CSR's 7n values
 * + indices.
 *   nx·ny·nz must equal the handle's n; with world > 1 rank r owns the planes
 *   [r·nz/world, (r+1)·nz/world) (nz % world == 0, else CCG_E_DIM), i.e. the
 *   same row range as every vector slice.
 *   coeffs : HOST double[8] = {Re d, Im d, Re ox, Im ox, Re oy, Im oy, Re oz, Im oz}
 *            (copied; finite, else CCG_E_ARG).
 *   flags  : unused (A is complex symmetric by construction).
 * Supports CCG_OP_A, CCG_OP_AT (= A) and CCG_OP_AH (conjugated coefficients),
 * hence every method, on any world size.
 *   Arithmetic: the terms are accumulated by FMA in ascending column order, as
 *   the CSR kernel does on the equivalent matrix; an omitted term is a zero
 *   coefficient times the point's own value, so the result equals the CSR
 *   product bit for bit except the sign of a component that underflowed to −0,
 *   and a non-finite u_i makes (A u)_i non-finite (as d·u_i already does).
 *   Off-diagonal coefficients with exactly zero imaginary parts (the
 *   Laplacian case) take a kernel that skips the multiplications by them. */
int ccg_set_matvec_stencil7(ccg_handle h, int64_t nx, int64_t ny, int64_t nz, const double* coeffs,
                            uint32_t flags);

/* FFT block-Toeplitz operator on an nx × ny × nz lattice (x fastest, global
 * index i = ix + nx·(iy + ny·iz), unit spacing):
 *   (A x)_i = d·x_i + Σ_{j≠i} K(r_i − r_j)·x_j,
 * the structure of the discrete-dipole systems CCGPAK was written for (P:47
 * [§1], DDSCAT; BASELINE configs 2 and 4 are scalar instances with
 * K(δ) = 0.1·exp(i k|δ|)/|δ|).  The product is a linear convolution computed
 * with the library's own 3-D FFT kernels on a power-of-two circulant
 * embedding: O(n log n) work and a few MB of traffic
 * instead of the dense n²·s bytes.  Aᵀ uses K(−δ), Aᴴ = conj(Aᵀ conj(x)).
 *   nx·ny·nz must equal the handle's n; each side in [1, 1024] (else CCG_E_DIM).
 *   kernel : HOST complex128 (interleaved doubles) K(δ) for every displacement
 *            δ = (dx, dy, dz), |dx| < nx, |dy| < ny, |dz| < nz, at index
 *            (dx + nx − 1) + (2nx − 1)·((dy + ny − 1) + (2ny − 1)·(dz + nz − 1));
 *            the δ = 0 entry is ignored.  Copied (transformed once, in double).
 *   diag   : HOST double[2] = {Re d, Im d}.
 *   flags  : informational (CCG_FLAG_SYMMETRIC if K(δ) = K(−δ)).
 * With world > 1 every rank transforms the gathered vector and keeps its own
 * rows (the FFT work is replicated; the vector is n·s bytes).  Supports
 * CCG_OP_A, CCG_OP_AH, CCG_OP_AT, hence every method.  Non-finite kernel or
 * diagonal values: CCG_E_ARG. */
int ccg_set_matvec_toeplitz3(ccg_handle h, int64_t nx, int64_t ny, int64_t nz, const double* kernel,
                             const double* diag, uint32_t flags);

/* User operator: the paper's own contract, P:95 [§5] "User can implement
 * his/her own sparse matrix scheme in matvec and cmatvec" (the product
 * is "separated from the conjugate gradient iterations itself").  The library
 * calls fn for every product and runs the iteration (fused vector passes,
 * reductions, scalar steps) around it.
 *   fn(user, op, x, y, n, row0, nloc, stream) must ENQUEUE on `stream` (a
 *   cudaStream_t) y[0:nloc] = (op(A)·x)[row0 : row0+nloc] and return 0, where
 *   op is CCG_OP_A / CCG_OP_AH / CCG_OP_AT, x a DEVICE pointer to the FULL
 *   length-n input (gathered over ranks when world > 1) and y a DEVICE pointer
 *   to nloc outputs, both in the handle's precision, valid only until the
 *   product's work completes on the stream.  A non-zero return aborts the
 *   call with CCG_E_USER.
 *   caps  : CCG_CB_A (required) | CCG_CB_AH | CCG_CB_AT — the products fn
 *           provides (methods needing Aᴴ without CCG_CB_AH: CCG_E_CAPABILITY);
 *           | CCG_CB_GRAPH_SAFE if fn only enqueues capturable asynchronous work
 *           (then the iteration runs as a replayed CUDA graph and fn is called
 *           once per method, at capture; otherwise fn is called every product).
 *   user  : opaque, passed back.  fn, user and whatever they reference are
 *           borrowed until ccg_destroy or the next set_matvec. */
enum { CCG_CB_A = 1, CCG_CB_AH = 2, CCG_CB_AT = 4, CCG_CB_GRAPH_SAFE = 8 };
typedef int (*ccg_matvec_fn)(void* user, int op, const void* x, void* y, int64_t n, int64_t row0,
                             int64_t nloc, void* stream);
int ccg_set_matvec_callback(ccg_handle h, ccg_matvec_fn fn, void* user, uint32_t caps, uint32_t flags);

/* y_local = (op(A)·x)[row0 : row0+nloc] from x_local = x[row0 : row0+nloc].
 * x_local / y_local may be HOST or DEVICE pointers (detected); nloc elements.
 * Collective over ranks.  Blocks until y_local is written. */
int ccg_apply(ccg_handle h, ccg_op op, const void* x_local, void* y_local);

/* Restart length m of CCG_GMRES (1 ≤ m ≤ 64, else CCG_E_ARG; default 30).  The
 * basis (m+1 vectors of nloc elements) is allocated by the next GMRES solve. */
int ccg_set_gmres_restart(ccg_handle h, int32_t m);

/* Right Jacobi preconditioning of the following ccg_solve calls (SURVEY §8(f)
 * NEXT-4): the method runs on B u = y with B = A·D⁻¹, D = diag(d), and returns
 * x = D⁻¹u.  The residual y − B u is the original y − A x, so tolerances and
 * the true residual keep their meaning; products by ccg_apply are unaffected.
 *   diag_local : HOST or DEVICE pointer to this rank's nloc diagonal entries d
 *                (the handle's precision; finite and nonzero, else CCG_E_ARG);
 *                copied.  NULL disables preconditioning.  Collective (world > 1).
 *   flags      : reserved, 0. */
int ccg_set_jacobi(ccg_handle h, const void* diag_local, uint32_t flags);

/* ℓ of CCG_BICGSTABL (1 ≤ ℓ ≤ 4, else CCG_E_ARG; default 2; ℓ = 1 is BiCGSTAB). */
int ccg_set_bicgstab_ell(ccg_handle h, int32_t ell);

/* Solve A x = y with `method` (stopping rule ‖r_k‖ ≤ tol·‖r_0‖
 * on the recurrence residual, r_0 = y − A·x0; true residual recomputed at exit).
 *   x0_local : initial guess slice (NULL => 0), y_local: right-hand side slice,
 *   x_local_out : solution slice.  HOST or DEVICE pointers (detected), nloc elements.
 *   tol ≥ 0 (epsilon_err), maxit ≥ 1.  tol = 0 runs exactly maxit iterations
 *   unless the recurrence residual is exactly 0 or a breakdown occurs.
 *   res : caller-owned, filled on CCG_OK.
 * Collective over ranks.  Blocks until the result is final. */
int ccg_solve(ccg_handle h, ccg_method method, const void* x0_local, const void* y_local,
              void* x_local_out, double tol, int32_t maxit, ccg_result* res);

/* Recurrence residual history ‖r_k‖/‖r_0‖, k = 0..iterations, of the last solve
 * (S:440-448).  Copies min(cap, available) doubles into rel_res (host), sets *len. */
int ccg_get_history(ccg_handle h, double* rel_res, int32_t cap, int32_t* len);

/* Device time of the matvec kernels of the last ccg_solve / ccg_apply when
 * timing is enabled (CUDA events on the handle's stream around every matvec
 * launch; disables graph capture and the single-cluster loop while on).
 * ms_a/ms_ah: summed milliseconds of the A·x and Aᴴ·x kernels (the QMR/BiCG
 * dual product counts as A·x); n_a/n_ah: products actually executed (launches
 * gated off after convergence are not counted, their few µs stay in the sum).
 * Any pointer may be NULL. */
int ccg_set_timing(ccg_handle h, int enable);
int ccg_get_timing(ccg_handle h, double* ms_a, int32_t* n_a, double* ms_ah, int32_t* n_ah);

/* Number of libccg kernel launches issued by the last ccg_solve / ccg_apply
 * (graph-launched kernels included; early-exit kernels after convergence
 * are counted because they are launched). */
int64_t ccg_last_launch_count(ccg_handle h);

/* Execution statistics of the last ccg_solve on this handle (diagnostics; the
 * evidence that the sharded data plane ran).  key:
 *   CCG_STAT_COMM_KIND          0 = no communicator, 1 = NCCL, 2 = loopback
 *   CCG_STAT_GRAPH_REPLAYS      iteration-graph launches (cudaGraphLaunch)
 *   CCG_STAT_GRAPH_COLLECTIVES  collective calls executed inside graph replays
 *                               (calls captured per iteration × replays)
 *   CCG_STAT_EAGER_COLLECTIVES  collective calls issued outside graphs (setup,
 *                               true residual, eager loops)
 *   CCG_STAT_WORLD, CCG_STAT_REPLICATED  the handle's world size / vector mode
 * Returns CCG_E_ARG for an unknown key or NULL value. */
enum { CCG_STAT_COMM_KIND = 0, CCG_STAT_GRAPH_REPLAYS = 1, CCG_STAT_GRAPH_COLLECTIVES = 2,
       CCG_STAT_EAGER_COLLECTIVES = 3, CCG_STAT_WORLD = 4, CCG_STAT_REPLICATED = 5,
       CCG_STAT_P2P_EXCHANGES = 6 /* P2P mirror exchanges issued (host side, since create) */,
       CCG_STAT_SYMMETRIC = 7 /* dense, one rank: 0 the general products, 1 upper-triangle products
                                 (CCG_FLAG_SYMMETRIC), 2 upper-triangle products, A = Aᵀ detected */ };
int ccg_get_stat(ccg_handle h, int32_t key, int64_t* value);

/* cudaStream_t of the handle (for callers that order their own work). */
void* ccg_get_stream(ccg_handle h);

/* Text of the last error on h (or of the last ccg_create failure if h is NULL).
 * Valid until the next call on h. */
const char* ccg_last_error(ccg_handle h);

int ccg_destroy(ccg_handle h);

/* Library version string "ccg-b200 <major>.<minor> sm_100a". */
const char* ccg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CCG_H_ */
