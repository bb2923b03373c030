// kernels.h — launchers of the sm_100a kernels of the solve path.
#pragma once
#include "psc_internal.h"

namespace psc {

// Row-wise sliced-ELL kernels: s_i = sum_k val * x[col] over row i (stored order,
// fused multiply-add), then an epilogue.  `x` is an owned+halo vector of the
// column space.  Reductions are deterministic: fixed warp-shuffle tree, fixed
// block order, finalised by the last CTA to finish (ticket), written to `red_out`.
enum class RowOp {
  Spmv,       // y = alpha s + beta y           (beta == 0: y not read)
  SpmvDot,    // y = s;  red0 += x_i * s        (q = A p and (p, q))
  Sweep,      // y = x_i + dinv_i (b_i - s)     (l1-Jacobi sweep, Jacobi: reads old x)
  SweepDot,   // Sweep, red0 += w_i * y_i, w = b unless RowArgs::w is set
              // (last level-0 post-sweep: (r, z) for PCG, (z, A p_old) for FCG)
  Resid,      // y = b_i - s
  ResidDot2,  // y = b_i - s; red0 += y_i^2; red1 += b_i^2
  PAdd,       // y += s                         (prolongation x_l += P x_{l+1})
  Sweep0,     // the first two l1-Jacobi sweeps from x = 0 in one pass:
              // y = x1_i + dinv_i (b_i - sum_j a_ij x1_j) with x1 = dinv .* b formed on
              // the fly (bit-identical to scale then Sweep); `x` is scratch, written
              // (x = x1) only by the two-launch fallback of non-TMA layouts
};

// Halo exchange folded into the producer ("fused push"): a row kernel
// whose output y is a halo-bearing vector stores each boundary row's value straight
// into the neighbours' halo slots (NVLink peer stores) from its epilogue, and its last
// CTA release-stores one generation flag per neighbour; the kernel that next reads
// y's halo waits for those flags before its first gather (WaitSpec).
struct PushSpec {
  int on = 0;
  int R = 0;
  const uint8_t* sslice = nullptr; // [n_own/32]: 1 if a row of the 32-row slice is sent
  const int32_t* iptr = nullptr;  // [n_own+1]: sends of owned row i at [iptr[i], iptr[i+1])
  const int32_t* iq = nullptr;    // peer of each send
  const int32_t* ipos = nullptr;  // slot in that peer's block of y's halo
  double* const* dst = nullptr;   // [R] peer p's halo slots for this rank's block of y
  const int32_t* nbr = nullptr;   // [R] neighbours at y's level
  uint64_t* const* pflag = nullptr;
  uint64_t* gen = nullptr;        // [R] signals sent to each peer (generation)
  unsigned int* ticket = nullptr;
};
struct WaitSpec {
  int on = 0;
  int R = 0;
  const int32_t* nbr = nullptr;   // [R] neighbours at x's level
  const uint64_t* myflag = nullptr;
  const uint64_t* gen = nullptr;  // wait until every neighbour's flag reaches my generation
  uint64_t timeout_ns = 0;
};

struct RowArgs {
  double alpha = 1.0, beta = 0.0;
  const double* x = nullptr;
  const double* b = nullptr;
  const double* dinv = nullptr;
  double* y = nullptr;
  double* y2 = nullptr;        // Spmv only: y2 = dinv2 .* y
  const double* dinv2 = nullptr;
  const double* w = nullptr;   // SweepDot only: weight of the reduction (nullptr: b)
  const RedSite* red = nullptr;
  double* red_out = nullptr;   // red0 -> red_out[0], red1 -> red_out[red_stride]
  int red_stride = 1;
  // all row vectors (b, dinv, x, y) are library buffers padded past n (TMA bulk
  // copies of the last chunk may read up to 8 bytes beyond the last row)
  bool vec_padded = false;
  PushSpec push;  // y's halo pushed by this kernel (push.on)
  WaitSpec wait;  // x's halo was pushed by the previous kernel: wait for it (wait.on)
};
// row kernels that implement PushSpec / WaitSpec (sliced ELL: TMA ring or plain)
bool rows_can_push(const Sell& A, const RowArgs& r);

// Which slices: all, interior only (no halo column), boundary only.
enum class SliceSet { All, Interior, Boundary };

int row_grid(const Sell& A, RowOp op, int num_sms, SliceSet set = SliceSet::All);
void launch_rows(psc_ctx* ctx, const Sell& A, RowOp op, const RowArgs& a, cudaStream_t s,
                 SliceSet set = SliceSet::All);

// x = dinv .* b  (first sweep from x = 0: x + M^-1 (b - A 0) = M^-1 b)
void launch_scale(psc_ctx* ctx, int64_t n, const double* dinv, const double* b, double* x, cudaStream_t s);
// m_i = a_ii + sum_{j != i} |a_ij| over the stored row;  dinv_i = 1 / m_i
void launch_l1_dinv(psc_ctx* ctx, const Sell& A, double* dinv, cudaStream_t s);
// gathered scalars: value of slot = sum over ranks of g[slot*nranks + r], in rank order
// CG: alpha = num / pq ; x += alpha p ; r -= alpha q ; red(r.r)
// num = sum of g_num[0..num_ranks-1] (PCG: rz_old, 1 entry; FCG: gathered (p, r))
void launch_cg_update(psc_ctx* ctx, int64_t n, double* x, const double* p, double* r, const double* q,
                      const double* g_pq, const double* g_num, int num_ranks, int nranks, const RedSite* red,
                      double* red_out, cudaStream_t s);
// FCG(1) direction: beta = (z, q_old) / (p_old, q_old) (both gathered); p = z - beta p; red(p.r)
void launch_fcg_dir(psc_ctx* ctx, int64_t n, const double* z, double* p, const double* r, const double* g_zq,
                    const double* g_pq, int nranks, const RedSite* red, double* red_out, cudaStream_t s);
// beta = rz / rz_old ; p = z + beta p ; then rz_old := rz (by the last CTA)
void launch_xpby(psc_ctx* ctx, int64_t n, const double* z, double* p, const double* g_rz, double* rz_old,
                 int nranks, const RedSite* red, cudaStream_t s);
// red(a . b)
void launch_dot(psc_ctx* ctx, int64_t n, const double* a, const double* b, const RedSite* red, double* red_out,
                cudaStream_t s);
// sendbuf[i] = x[idx[i]]
void launch_pack(psc_ctx* ctx, int64_t n, const int32_t* idx, const double* x, double* sendbuf, cudaStream_t s);
// out[i] = in[map[i]]  (gather from a replicated vector into owned+halo layout)
void launch_gather(psc_ctx* ctx, int64_t n, const int64_t* map, const double* in, double* out, cudaStream_t s);
// Coarsest solver in ONE CTA: x = dinv .* b, then nsweeps-1 l1-Jacobi sweeps in shared memory.
// Requires n <= coarse_smem_rows().
int64_t coarse_smem_rows();
bool coarse_one_cta_fits(const Sell& A);  // A_coarse fits the one-CTA solver's shared memory
void launch_coarse_solve(psc_ctx* ctx, const Sell& A, const double* dinv, const double* b, double* x, int nsweeps,
                         cudaStream_t s);

// Dense coarsest solver (n <= coarse_dense_max_rows()): dense = row-major n x n copy of A.
int64_t coarse_dense_max_rows();
void dense_from_sell(psc_ctx* ctx, const Sell& A, double* dense, cudaStream_t s);
void launch_coarse_dense(psc_ctx* ctx, const double* dense, int64_t n, const double* dinv, const double* b, double* x,
                         int nsweeps, cudaStream_t s);

// Coarsest-level PCG with the l1-Jacobi preconditioner, dense one-CTA form:
// x = PCG(A, b) from zero, at most maxit iterations, stop when ||r|| <= tol ||b||.
void launch_coarse_dense_pcg(psc_ctx* ctx, const double* dense, int64_t n, const double* dinv, const double* b,
                             double* x, int maxit, double tol, cudaStream_t s);
// ... and its general (launch-per-step) form; scalars are gathered partials
// (nr entries each, summed in rank order), `done` a device stop flag:
//   init:   x = 0, r = b, z = dinv r, p = z; red (r, z) -> out[0], (b, b) -> out[stride]; done = 0
//   update: if !done: pq = (p, q); pq <= 0: done; else alpha = rz / pq, x += alpha p,
//           r -= alpha q, z = dinv r; red (r, r) -> out[0], (r, z) -> out[stride]
//   dir:    if !done: ||r|| <= tol ||b||: done; else p = z + (rz_new / rz) p
void launch_cpcg_init(psc_ctx* ctx, int64_t n, const double* b, const double* dinv, double* x, double* r, double* z,
                      double* p, int* done, const RedSite* red, double* out, int stride, cudaStream_t s);
void launch_cpcg_update(psc_ctx* ctx, int64_t n, double* x, const double* p, double* r, const double* q, double* z,
                        const double* dinv, const double* g_pq, const double* g_rz, int nr, int* done,
                        const RedSite* red, double* out, int stride, cudaStream_t s);
void launch_cpcg_dir(psc_ctx* ctx, int64_t n, const double* z, double* p, const double* g_rr, const double* g_bb,
                     const double* g_rzn, const double* g_rz, int nr, double tol, int* done, cudaStream_t s);

// y = D b, D dense row-major n x n (n <= dense_gemv_max_rows()); out = in^T (n x n)
int64_t dense_gemv_max_rows();
void launch_dense_gemv(psc_ctx* ctx, const double* D, int64_t n, const double* b, double* y, cudaStream_t s);
void launch_transpose(psc_ctx* ctx, const double* in, int64_t n, double* out, cudaStream_t s);

// CSR (global int64 columns) -> sliced ELL with local int32 columns.
// lanes: 0 = choose from the mean row length (choose_lanes), else 1 / 4 / 8 / 16 / 32.
int choose_lanes(int64_t n_rows, int64_t nnz);
void sell_from_csr(psc_ctx* ctx, int64_t n_rows, const int64_t* d_rowptr, const int64_t* d_colg,
                   const double* d_val, int64_t nnz, int64_t own_begin, int64_t n_own, const int64_t* d_halo,
                   int64_t n_halo, Sell& S, cudaStream_t s, int lanes = 0, bool allow_dia = false);
void sell_free(Sell& S);
// new values in the CSR order of the assembled matrix (device array of S.nnz)
void sell_update_values(psc_ctx* ctx, Sell& S, const double* d_newval, cudaStream_t s);

RedSite red_alloc(int num_sms, int nred);
void red_free(RedSite& r);

}  // namespace psc
