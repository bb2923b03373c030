/* psc.h — C ABI of the B200-native AMG-PCG solve phase (libpsc.so).
 *
 * The method is the solve phase of PSCToolkit (arXiv 2406.19754, PAPER.md):
 * FP64 preconditioned conjugate gradient on a row-block-distributed SPD sparse
 * matrix, preconditioned by one AMG V-cycle per iteration (Eq. (2), P:202-207,
 * Sec. 2.3) over a GIVEN aggregation hierarchy {A_l, P_l, R_l = P_l^T}, with
 * l1-Jacobi pre/post-smoothing (Sec. 2.3.2) and a fixed number of
 * l1-Jacobi sweeps at the coarsest level (Fig. 5 caption).
 *
 * The call order follows the paper's statement of a PSBLAS application
 * (Sec. 2.1): initialise the parallel + accelerator environment
 * (psb_init / psb_cuda_init), create the index-space descriptors (psb_cdall),
 * insert the matrices in GLOBAL numbering (psb_spall / psb_spins), assemble the
 * descriptors (psb_cdasb: halo lists) and the matrices (psb_spasb with the GPU
 * "mold": here a device sliced-ELL), build the preconditioner (the smoother
 * build of P:164-166: the l1 diagonals), and call the Krylov solver
 * (psb_krylov, Fig. 6) with x holding the initial guess on entry.
 *
 *   psc_init -> psc_desc_create (one per level index space)
 *            -> psc_mat_create_csr (A_l: rows l, cols l; P_l: rows l, cols l+1;
 *                                   R_l: rows l+1, cols l)
 *            -> psc_desc_assemble (each) -> psc_mat_assemble (each)
 *            -> psc_hier_create -> psc_pcg_solve ... -> destroy in reverse order.
 *
 * CONVENTIONS
 *  - Return value: int status.  PSC_OK (0); PSC_NOT_CONVERGED (1, psc_pcg_solve*
 *    only; outputs are valid); negative = error (mirrors PSBLAS `info`,
 *    P:105-107).  psc_last_error(ctx) gives a message for the last error.
 *  - Global indices are int64 ("8-byte integers for extreme-scale problems",
 *    P:62-63).  Device-local indices are int32 (owned first, then halo).
 *  - Ownership is a contiguous block partition: rank r owns global rows
 *    [row_start[r], row_start[r+1]) of an index space; row_start is identical on
 *    all ranks, starts at 0, is non-decreasing and ends at n_global.
 *  - CSR input: row_ptr[0] = 0, non-decreasing; columns strictly increasing
 *    within a row; 0 <= column < n_global(col space).  Violations: PSC_ERR_ARG.
 *  - Memory: the library copies every host array it is given at *_create*; the
 *    caller keeps its arrays.  Vector arguments named *_dev are device pointers to
 *    contiguous FP64 arrays on the context's GPU (e.g. torch.Tensor.data_ptr()),
 *    of length n_owned of the relevant index space; they belong to the caller.
 *    Arguments named *_host are host pointers.
 *  - Streams: all work runs on the library's own stream, ordered after the work
 *    already submitted to the `user_stream` given at psc_init (NULL = legacy
 *    default stream); every call returns after its GPU work is complete.
 *  - Collective: calls marked [collective] must be issued by every rank in the
 *    same order.  One host thread per context.
 *  - No CPU fallback: every numerical step runs in this library's CUDA kernels
 *    (sm_100a) and NCCL; a missing GPU is PSC_ERR_CUDA.
 */
#ifndef PSC_H
#define PSC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSC_OK 0
#define PSC_NOT_CONVERGED 1
#define PSC_ERR_ARG (-1)       /* bad argument / dimension mismatch / malformed CSR */
#define PSC_ERR_STATE (-2)     /* wrong call order: unassembled object, missing level */
#define PSC_ERR_CUDA (-3)      /* CUDA runtime error (including: no device) */
#define PSC_ERR_NCCL (-4)      /* NCCL error */
#define PSC_ERR_NOMEM (-5)     /* device or host allocation failed */
#define PSC_ERR_BREAKDOWN (-6) /* PCG: p^T A p <= 0 or not finite */

typedef struct psc_ctx_s psc_ctx;
typedef struct psc_desc_s psc_desc;
typedef struct psc_mat_s psc_mat;
typedef struct psc_hier_s psc_hier;

/* ------------------------------------------------------------------ context */

/* Fill id[128] with a fresh NCCL unique id.  Call on rank 0 only and broadcast
 * the bytes to the other ranks (e.g. with torch.distributed) before psc_init. */
int psc_get_unique_id(unsigned char id[128]);

/* Parallel + accelerator environment (psb_init + psb_cuda_init).
 * [collective when nranks > 1]  rank in [0, nranks); cuda_device = device
 * ordinal; id = 128 bytes from psc_get_unique_id (ignored, may be NULL, when
 * nranks == 1); user_stream = cudaStream_t the caller's producers/consumers use
 * (may be NULL).  On success *ctx owns a CUDA stream and (nranks > 1) an NCCL
 * communicator. */
int psc_init(int rank, int nranks, int cuda_device, const unsigned char* id, void* user_stream, psc_ctx** ctx);
void psc_finalize(psc_ctx* ctx);
const char* psc_status_string(int status);
const char* psc_last_error(psc_ctx* ctx);
/* Library build string (compiler, arch). */
const char* psc_version(void);
/* The cudaStream_t all of this context's work runs on (for callers that bracket
 * library calls with their own CUDA events).  Owned by the context. */
void* psc_ctx_stream(psc_ctx* ctx);

/* --------------------------------------------------------------- descriptor */

/* Index space of n_global entries split in contiguous row blocks (psb_cdall,
 * P:81-86; Fig. 1).  row_start: host, nranks+1 entries, copied. */
int psc_desc_create(psc_ctx* ctx, int64_t n_global, const int64_t* row_start, psc_desc** d);

/* [collective] Build halo lists (psb_cdasb): the halo of this index space is
 * the sorted set of off-rank global indices referenced by the columns of every
 * matrix created with this descriptor as `cols`; local numbering is owned
 * [0, n_owned) then halo [n_owned, n_owned + n_halo) ordered by global index
 * (hence grouped by owner).  Send lists are negotiated with the owners.  All
 * matrices whose columns live in this space must be created before this call. */
int psc_desc_assemble(psc_desc* d);

/* After assembly: n_owned, n_halo, first owned global index (any may be NULL). */
int psc_desc_info(psc_desc* d, int64_t* n_owned, int64_t* n_halo, int64_t* own_begin);
/* Test hook: halo_globals_host[n_halo] = global index of each halo slot. */
int psc_desc_halo(psc_desc* d, int64_t* halo_globals_host);
void psc_desc_destroy(psc_desc* d);

/* Host-only halo planning (no GPU, no NCCL), the arithmetic of psc_desc_assemble:
 * refs[n_refs] = global columns referenced by this rank's rows (any order,
 * duplicates allowed).  Writes the sorted unique off-rank ones to halo (capacity
 * n_refs) and their count to *n_halo, and recv_count[nranks] = halo entries owned
 * by each rank (the requests this rank sends to each owner, in halo order).
 * Errors: PSC_ERR_ARG for a malformed partition or an out-of-range column. */
int psc_halo_plan(int nranks, int rank, const int64_t* row_start, int64_t n_refs, const int64_t* refs, int64_t* halo,
                  int64_t* n_halo, int64_t* recv_count);
/* Host-only: local (owned) indices to send, for the requests received from the
 * peers: requests = the peers' halo lists for this rank, concatenated in peer
 * order, send_count[nranks] their lengths.  send_idx[sum send_count] (int32).
 * PSC_ERR_STATE if a request is not owned by this rank. */
int psc_send_plan(int nranks, int rank, const int64_t* row_start, const int64_t* send_count, const int64_t* requests,
                  int32_t* send_idx);

/* ------------------------------------------------------------------- matrix */

/* Insert this rank's rows of a distributed matrix in GLOBAL numbering (psb_spall
 * + psb_spins).  rows/cols: descriptors of the row and column index
 * spaces; n_local_rows must equal rows' owned count; row_ptr[n_local_rows+1]
 * (int64, local rows), col_global[nnz] (int64), val[nnz] (f64): host arrays,
 * copied to the device.  Off-rank columns are registered as halo of `cols`. */
int psc_mat_create_csr(psc_ctx* ctx, psc_desc* rows, psc_desc* cols, int64_t n_local_rows, const int64_t* row_ptr,
                       const int64_t* col_global, const double* val, psc_mat** m);

/* Renumber columns to local (owned then halo) and convert the device CSR into the
 * device sliced-ELL format (Hacked ELLPACK of P:168-183: 32-row slices, each its
 * own column-major ELLPACK block, padding value 0.0 with the row's last valid
 * column).  Needs both descriptors assembled. */
int psc_mat_assemble(psc_mat* m);

/* After assembly (any pointer may be NULL): nnz stored; padded = total device slots
 * including padding; n_units = warp work units (32-row slices, or 32/lanes-row
 * blocks); n_rows local rows; lanes = 1 for the sliced-ELL layout (one thread per
 * row), or G in {4, 8, 16, 32} for the row-group layout (G lanes per row, rows
 * padded to multiples of G) chosen for long rows. */
int psc_mat_info(psc_mat* m, int64_t* nnz, int64_t* padded, int64_t* n_units, int64_t* n_rows, int* lanes);

/* [collective] y_dev = alpha * A * x_dev + beta * y_dev (test hook; includes the
 * halo exchange of x).  x_dev: n_owned(cols); y_dev: n_owned(rows). */
int psc_mat_spmv(psc_mat* m, double alpha, const double* x_dev, double beta, double* y_dev);
void psc_mat_destroy(psc_mat* m);

/* -------------------------------------------------------------- hierarchy */

/* Coarsest-level solver B_ell of Eq. (2). */
enum {
  PSC_COARSE_SWEEPS = 0, /* coarse_sweeps l1-Jacobi sweeps from zero (Fig. 5 caption) */
  PSC_COARSE_PCG = 1     /* PCG from zero with the l1-Jacobi preconditioner, at most coarse_maxit
                            iterations, stopping when ||r||_2 <= coarse_tol ||b||_2 (the paper's
                            VBM configuration; reading R23).  The preconditioner B then
                            varies between applications: use PSC_KRYLOV_FCG. */
};

/* Smoothing sweeps before / after the coarse correction and the coarsest-level
 * solver (defaults 4 / 4 / 30 sweeps: Fig. 5 caption).  Zero-
 * initialise the struct: coarse_solver 0 = sweeps; coarse_maxit 0 -> 40 and
 * coarse_tol 0 -> 1e-10 (defaults of PSC_COARSE_PCG, reading R23).
 * variable_v 1 = variable V-cycle (VMATCH, P:330 footnote: "2 smoother iteration
 * at the first level, and doubled at each following level"): level l < L-1 runs
 * pre_sweeps*2^l / post_sweeps*2^l sweeps (reading R25); the coarsest solver is
 * unchanged.  PSC_ERR_ARG when a level would need more than 2^20 sweeps. */
typedef struct {
  int pre_sweeps;
  int post_sweeps;
  int coarse_sweeps;
  int coarse_solver;  /* PSC_COARSE_SWEEPS or PSC_COARSE_PCG */
  int coarse_maxit;
  double coarse_tol;
  int variable_v;     /* 0 = V-cycle, 1 = variable V-cycle (P:330 footnote) */
  int smoother;       /* PSC_SMOOTHER_L1JACOBI (0) or PSC_SMOOTHER_AINV (1) on the levels < L-1 */
  double ainv_drop;   /* AINV drop tolerance (entries |z_kj| < ainv_drop dropped; reading R27) */
} psc_cycle_opts;

/* Smoothers (Sec. 2.3.2).  AINV: M^-1 = Z D^-1 Z^T from an incomplete
 * A-biconjugation of A_l (W = Z for SPD A, reading R27), built on the host from the
 * matrix's host copy and applied on the device as two SpMVs (Z^T, then Z): a sweep
 * is r = b - A x, u = D^-1 Z^T r, x += Z u.  One rank (the paper's block-Jacobi form
 * across ranks is not built: PSC_ERR_STATE). */
enum { PSC_SMOOTHER_L1JACOBI = 0, PSC_SMOOTHER_AINV = 1 };

/* [collective] AMG hierarchy handle over given level matrices (D10/D11 in
 * SURVEY.md): A[0..nlevels-1], P[0..nlevels-2], R[0..nlevels-2] (R_l = P_l^T given
 * explicitly).  Builds the l1-Jacobi smoothers M_l = diag(A_l) + diag(sum_{j!=i}
 * |a_ij|) (the smoother-build step of P:164-166) and the device
 * workspace.  opts NULL = defaults.  Matrices must stay alive until
 * psc_hier_destroy. */
int psc_hier_create(psc_ctx* ctx, int nlevels, psc_mat* const* A, psc_mat* const* P, psc_mat* const* R,
                    const psc_cycle_opts* opts, psc_hier** h);

/* Local sizes: n_owned[l], nnz of A_l, P_l, R_l on this rank (arrays of nlevels; any may be NULL). */
int psc_hier_info(psc_hier* h, int* nlevels, int64_t* n_owned, int64_t* nnz_A, int64_t* nnz_P, int64_t* nnz_R);

/* [collective] z_dev = B_0 r_dev: one V-cycle (Eq. (2)) from zero. */
int psc_hier_vcycle(psc_hier* h, const double* r_dev, double* z_dev);

/* Test hook: dinv_dev[n_owned(level)] = 1 / M_level (the stored reciprocal l1 diagonal). */
int psc_hier_dinv(psc_hier* h, int level, double* dinv_dev);

/* [collective] Test hook: x_dev = nsweeps l1-Jacobi sweeps x <- x + M^{-1}(b - A_l x)
 * from x = 0 at `level` (sweeps at every level, whatever the coarse_solver option). */
int psc_hier_smooth(psc_hier* h, int level, const double* b_dev, double* x_dev, int nsweeps);

/* Solve statistics. */
typedef struct {
  int iters;                    /* PCG iterations performed */
  int status;                   /* same as the return value */
  double rel_res;               /* ||r_k||_2 / ||b||_2 at exit (recurrence residual) */
  double solve_seconds;         /* device time of the solve (CUDA events on the library stream) */
  int64_t kernel_launches;      /* library kernels launched during the solve */
  int64_t collectives;          /* NCCL calls issued during the solve */
  double dom_kernel_seconds;    /* summed device time of the level-0 l1-Jacobi sweep launches */
  int64_t dom_kernel_launches;  /* number of those launches */
  double dom_kernel_bytes;      /* algorithmic bytes per launch: 8 nnz(A_0) + 4 nnz_ell(A_0) + 32 n_0 */
  int64_t h2d_bytes, d2h_bytes; /* host<->device bytes moved by psc_pcg_solve_host */
  int halo_path;                /* 0 single rank, 1 NVLink peer stores (CUDA IPC), 2 NCCL */
  int iter_graph_nodes;         /* kernel launches per PCG iteration (captured graph) */
  int dom_kernel_per_iter;      /* level-0 sweep launches per Krylov iteration ((pre-1) + post) */
} psc_stats;

/* [collective] PCG (reading R1 of DESIGN.md) preconditioned by one
 * V-cycle per iteration.  b_dev: RHS; x_dev: initial guess on entry, solution on
 * exit (Fig. 6 caption); both n_owned(level 0), device.  Stops when
 * ||r_k||_2/||b||_2 <= tol (recurrence residual) or after maxit iterations.
 * res_hist_host: NULL or >= maxit+1 doubles, receives ||r_k||/||b|| for k = 0..iters.
 * st: NULL or receives statistics.  Returns PSC_OK, PSC_NOT_CONVERGED or an error
 * (PSC_ERR_BREAKDOWN when p^T A p <= 0 or non-finite).  b = 0 gives x = 0 and 0
 * iterations. */
int psc_pcg_solve(psc_hier* h, const double* b_dev, double* x_dev, double tol, int maxit, double* res_hist_host,
                  psc_stats* st);

/* [collective] Same, with HOST b and x (n_owned(0) each): the host->device copy of b
 * and x0 and the device->host copy of x are inside the call (end-to-end path). */
int psc_pcg_solve_host(psc_hier* h, const double* b_host, double* x_host, double tol, int maxit,
                       double* res_hist_host, psc_stats* st);

/* Krylov method of psc_krylov_solve ("a synchronization-reduced version of
 * the Flexible Conjugate Gradient (FCG)"; Fig. 6). */
enum {
  PSC_KRYLOV_PCG = 0, /* as psc_pcg_solve */
  PSC_KRYLOV_FCG = 1  /* Notay's FCG(1): z = B r; p = z - ((z, A p_old)/(p_old, A p_old)) p_old;
                         alpha = (p, r)/(p, A p).  Equal to PCG in exact arithmetic for a fixed
                         SPD B; stays convergent when B varies (PSC_COARSE_PCG).  Same stopping
                         rule, history, statistics and status codes as PCG. */
};

/* [collective] psc_pcg_solve / psc_pcg_solve_host with the Krylov method chosen by
 * `method` (PSC_KRYLOV_PCG or PSC_KRYLOV_FCG; anything else is PSC_ERR_ARG).
 * b, x: device (psc_krylov_solve) or host (psc_krylov_solve_host) buffers of
 * n_owned(0) doubles, x holding the initial guess on entry. */
int psc_krylov_solve(psc_hier* h, int method, const double* b_dev, double* x_dev, double tol, int maxit,
                     double* res_hist_host, psc_stats* st);
int psc_krylov_solve_host(psc_hier* h, int method, const double* b_host, double* x_host, double tol, int maxit,
                          double* res_hist_host, psc_stats* st);

/* [collective] Timing hook: *us_per_exchange = device time of one halo exchange of a
 * level-`level` vector, averaged over `reps` back-to-back exchanges (eager launches). */
int psc_hier_exchange_bench(psc_hier* h, int level, int reps, double* us_per_exchange);

/* One kernel (name, hierarchy level) of the Krylov iteration, as measured by
 * psc_hier_kernel_profile.  level: hierarchy level of a V-cycle kernel, -1 for the
 * Krylov-level kernels (q = A p, vector updates, exchanges of p).  Bytes per call:
 * alg_bytes = SURVEY.md §8(d)'s algorithmic count (12 B per stored nonzero + 8 B per
 * vector element read or written once); layout_bytes = the same vectors + the matrix
 * as stored (value and column slots incl. padding, slice headers, row order). */
typedef struct {
  char name[64];       /* kernel family and epilogue, e.g. "sell_tma<Sweep>" */
  int level;
  int calls_per_iter;  /* launches of this (name, level) per Krylov iteration */
  double total_us;     /* device time of those launches per iteration (event pairs) */
  double alg_bytes, layout_bytes;  /* per call */
} psc_kernel_rec;

/* [collective] Per-kernel device timing: solves A x = b from x = 0
 * for exactly `iters` iterations (no tolerance test; b on the device, n_owned(0))
 * with a CUDA graph of one iteration in which every kernel launch is bracketed by
 * an event pair, and returns up to max_recs records (grouped by name and level, in
 * launch order) and their number in *n_recs.  The caller's b is not modified; the
 * iterate is discarded.  Errors: PSC_ERR_ARG (iters < 1, null pointers, unknown
 * method), PSC_ERR_BREAKDOWN. */
int psc_hier_kernel_profile(psc_hier* h, int method, const double* b_dev, int iters, psc_kernel_rec* recs,
                            int max_recs, int* n_recs);

void psc_hier_destroy(psc_hier* h);

/* Structure-preserving coefficient update ("interfaces that allow to update
 * data coefficients in an existing matrix if the structure is preserved"): val_host
 * holds nnz values in the CSR order the matrix was created with (same row_ptr and
 * columns).  Before assembly the staged values are replaced; after assembly the
 * device sliced-ELL values (and the host copy, if kept) are.  Hierarchies using the
 * matrix see the new values at their next kernel; their smoothers do not change until
 * psc_hier_rebuild_smoothers.  Errors: PSC_ERR_ARG. */
int psc_mat_update_values(psc_mat* m, const double* val_host);

/* [collective] Rebuild every level's smoother from the current values of A_l (the
 * second step of the split build: "the construction of the smoothers ...
 * can be executed multiple times reusing an already assembled hierarchy"): l1
 * diagonals, AINV factors, the dense coarsest copy and the dense suffix operator; the
 * hierarchy (A_l, P_l, R_l) is reused as it is.  A replicated coarse suffix (several
 * ranks) keeps its copies: PSC_ERR_STATE. */
int psc_hier_rebuild_smoothers(psc_hier* h);

/* ---------------------------------------------------------------------------------
 * AMG set-up on the device.  The paper builds
 * the hierarchy "mostly on the CPU side" and names GPU set-up as future
 * work; here every step runs in CUDA kernels on ctx's device:
 *   decoupled Vanek-Mandel-Brezina aggregation, strong set N_i(theta) =
 *     {j != i : |a_ij| >= theta sqrt(a_ii a_jj)} (phase 1 = the VMB root rule
 *     in increasing index, computed in parallel rounds (reading R26); phase 2 = the
 *     strongest strong neighbour's aggregate (R18));
 *   tentative prolongator of Eq. (3) with w = 1, smoothed
 *     P = (I - omega D^-1 A) P^, omega = 1/||D^-1 A||_inf;
 *   R = P^T; Galerkin A_{l+1} = R A_l P;
 *   stop when n_l <= coarse_target, at max_levels, or when aggregation would keep
 *     more than stall_ratio n_l nodes (R19).
 * Each value is computed in the order the definitions state with one IEEE rounding per
 * operation (no FMA contraction), so a sequential implementation reproduces it bit
 * for bit. */
typedef struct psc_amg_s psc_amg;
typedef struct {
  double theta;           /* strength threshold (R17: 0.01) */
  int max_levels;         /* 20 */
  int64_t coarse_target;  /* 200 */
  double stall_ratio;     /* 0.75 */
} psc_amg_opts;

/* [one rank] Build the hierarchy of A_0 (n x n, host CSR: int64 row_ptr[n+1], int64
 * col (strictly increasing per row, in [0, n)), f64 val; copied, the caller keeps
 * its arrays).  opts may be NULL (defaults above).  Errors: PSC_ERR_ARG (malformed
 * CSR, a row without a positive diagonal, bad options), PSC_ERR_STATE (nranks > 1),
 * PSC_ERR_CUDA / PSC_ERR_NOMEM. */
int psc_amg_build(psc_ctx* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                  const psc_amg_opts* opts, psc_amg** out);
/* Sizes and timings.  Arrays (each may be NULL) hold >= *nlevels entries: rows,
 * nnz(A_l), nnz(P_l) (0 at the coarsest), omega_l, phase-1 rounds; seconds[5] =
 * aggregation, prolongator, transpose, Galerkin, total (host wall clock around the
 * device work, synchronised). */
int psc_amg_info(psc_amg* a, int* nlevels, int64_t* n, int64_t* nnz_A, int64_t* nnz_P, double* omega,
                 int* mis_rounds, double* seconds);
/* Copy level `level`'s matrix (kind 0 = A_l, 1 = P_l, 2 = R_l; P/R absent at the
 * coarsest level: PSC_ERR_STATE) to host arrays sized from psc_amg_info (row_ptr:
 * rows + 1; col, val: nnz).  Any pointer may be NULL. */
int psc_amg_level_csr(psc_amg* a, int level, int kind, int64_t* row_ptr, int64_t* col, double* val);
/* Aggregate of each node of level `level` (< nlevels - 1) and its root flags (1 = root). */
int psc_amg_aggregates(psc_amg* a, int level, int64_t* agg, int8_t* root);
/* Descriptors, assembled matrices and psc_hier_create over the set-up's levels
 * (once per set-up).  The hierarchy uses matrices owned by `a`: destroy it before
 * psc_amg_destroy. */
int psc_amg_hier_create(psc_amg* a, const psc_cycle_opts* opts, psc_hier** out);
void psc_amg_destroy(psc_amg* a);

#ifdef __cplusplus
}
#endif
#endif /* PSC_H */
