// kernels.cu — sm_100a kernels of the AMG-PCG solve path (FP64, CUDA cores).
//
// Nothing on this path is a dense contraction ("arithmetic intensity is
// of order O(1) ... memory/communication-bound"), so there are no tensor-core
// ops: every kernel is written for HBM bandwidth — coalesced 8-byte per-lane
// streams of the sliced-ELL values/columns (evict-first, __ldcs), read-only
// cached gathers of x (__ldg, kept in the 126 MB L2), grid-stride loops sized
// to the SM count, and deterministic fixed-order reductions.
#include <cub/cub.cuh>

#include "kernels.h"

namespace psc {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double gsum(const double* g, int nranks) {
  // value of a gathered scalar: sum over ranks in rank order (identical on all ranks)
  double s = 0.0;
  for (int r = 0; r < nranks; ++r) s += __ldcg(g + r);
  return s;
}

// Deterministic block + grid reduction of NR values.  Every CTA writes its
// partials; the CTA that draws the last ticket sums all partials in a fixed
// order and writes out[j * out_stride].
template <int NR>
__device__ __forceinline__ void grid_reduce(double (&acc)[NR], double* partials, unsigned int* ticket,
                                            double* out, int out_stride) {
  __shared__ double sm[NR][32];
  __shared__ bool am_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    double v = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sm[j][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      double t = 0.0;
      for (int w = 0; w < nwarp; ++w) t += sm[j][w];
      partials[j * gridDim.x + blockIdx.x] = t;
    }
    __threadfence();
    unsigned int tk = atomicAdd(ticket, 1u);
    am_last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    double v = 0.0;
    for (unsigned int i = threadIdx.x; i < gridDim.x; i += blockDim.x) v += __ldcg(partials + j * gridDim.x + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) sm[j][warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nwarp; ++w) t += sm[j][w];
      out[j * out_stride] = t;
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// Row sum of `lane`'s row in slice s: s = sum_k val[k] * x[col[k]], k in stored
// order (padding contributes fma(0, x, s) = s).  Loads of a batch of up to 8
// (value, column) pairs are issued before the dependent gathers for memory-level
// parallelism.
__device__ __forceinline__ double sell_row_sum(const int64_t* __restrict__ sptr, const int32_t* __restrict__ col,
                                               const double* __restrict__ val, int64_t s, int lane,
                                               const double* __restrict__ x) {
  const int64_t b = sptr[s];
  const int w = (int)((sptr[s + 1] - b) >> 5);
  const int32_t* c = col + b + lane;
  const double* v = val + b + lane;
  double sum = 0.0;
  int k = 0;
  for (; k + 8 <= w; k += 8) {
    int ci[8];
    double vi[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      ci[j] = __ldcs(c + 32 * j);
      vi[j] = __ldcs(v + 32 * j);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) sum = fma(vi[j], __ldg(x + ci[j]), sum);
    c += 256;
    v += 256;
  }
  const int rem = w - k;
  if (rem > 0) {
    int ci[8];
    double vi[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < rem) {
        ci[j] = __ldcs(c + 32 * j);
        vi[j] = __ldcs(v + 32 * j);
      }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < rem) sum = fma(vi[j], __ldg(x + ci[j]), sum);
  }
  return sum;
}

struct RowKArgs {
  const int64_t* sptr;
  const int32_t* col;
  const double* val;
  const int32_t* list;  // nullptr: slices 0..nlist-1
  int64_t nlist;
  int64_t n_rows;
  double alpha, beta;
  const double* x;
  const double* b;
  const double* dinv;
  double* y;
  double* partials;
  unsigned int* ticket;
  double* red_out;
  int red_stride;
};

template <RowOp OP>
__global__ void __launch_bounds__(kBlock) row_kernel(RowKArgs a) {
  constexpr int NR = (OP == RowOp::SpmvDot || OP == RowOp::SweepDot) ? 1 : (OP == RowOp::ResidDot2 ? 2 : 0);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * kWarpsPerBlock;
  double acc[NR > 0 ? NR : 1] = {};
  for (int64_t t = (int64_t)blockIdx.x * kWarpsPerBlock + warp; t < a.nlist; t += stride) {
    const int64_t s = a.list ? (int64_t)a.list[t] : t;
    const double sum = sell_row_sum(a.sptr, a.col, a.val, s, lane, a.x);
    const int64_t i = s * kSlice + lane;
    if (i < a.n_rows) {
      if constexpr (OP == RowOp::Spmv) {
        a.y[i] = (a.beta == 0.0) ? a.alpha * sum : a.alpha * sum + a.beta * a.y[i];
      } else if constexpr (OP == RowOp::SpmvDot) {
        a.y[i] = sum;
        acc[0] += a.x[i] * sum;
      } else if constexpr (OP == RowOp::Sweep || OP == RowOp::SweepDot) {
        const double bi = a.b[i];
        const double xn = a.x[i] + a.dinv[i] * (bi - sum);
        a.y[i] = xn;
        if constexpr (OP == RowOp::SweepDot) acc[0] += bi * xn;
      } else if constexpr (OP == RowOp::Resid) {
        a.y[i] = a.b[i] - sum;
      } else if constexpr (OP == RowOp::ResidDot2) {
        const double bi = a.b[i];
        const double r = bi - sum;
        a.y[i] = r;
        acc[0] += r * r;
        acc[1] += bi * bi;
      } else if constexpr (OP == RowOp::PAdd) {
        a.y[i] += sum;
      }
    }
  }
  if constexpr (NR > 0) grid_reduce<NR>(acc, a.partials, a.ticket, a.red_out, a.red_stride);
}

template <RowOp OP>
static int occupancy_blocks() {
  static int occ = -1;
  if (occ < 0) {
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, row_kernel<OP>, kBlock, 0) != cudaSuccess || o < 1) o = 1;
    occ = o;
  }
  return occ;
}

static int occ_for(RowOp op) {
  switch (op) {
    case RowOp::Spmv: return occupancy_blocks<RowOp::Spmv>();
    case RowOp::SpmvDot: return occupancy_blocks<RowOp::SpmvDot>();
    case RowOp::Sweep: return occupancy_blocks<RowOp::Sweep>();
    case RowOp::SweepDot: return occupancy_blocks<RowOp::SweepDot>();
    case RowOp::Resid: return occupancy_blocks<RowOp::Resid>();
    case RowOp::ResidDot2: return occupancy_blocks<RowOp::ResidDot2>();
    case RowOp::PAdd: return occupancy_blocks<RowOp::PAdd>();
  }
  return 1;
}

static int64_t set_count(const Sell& A, SliceSet set) {
  return set == SliceSet::All ? A.n_slices : (set == SliceSet::Interior ? A.n_interior : A.n_boundary);
}

int row_grid(const Sell& A, RowOp op, int num_sms, SliceSet set) {
  const int64_t n = set_count(A, set);
  const int64_t need = (n + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int64_t cap = (int64_t)num_sms * occ_for(op);
  return (int)std::max<int64_t>(1, std::min(need, cap));
}

void launch_rows(psc_ctx* ctx, const Sell& A, RowOp op, const RowArgs& r, cudaStream_t s, SliceSet set) {
  RowKArgs a;
  a.sptr = A.slice_ptr;
  a.col = A.col;
  a.val = A.val;
  a.list = set == SliceSet::All ? nullptr : (set == SliceSet::Interior ? A.interior : A.boundary);
  a.nlist = set_count(A, set);
  a.n_rows = A.n_rows;
  a.alpha = r.alpha;
  a.beta = r.beta;
  a.x = r.x;
  a.b = r.b;
  a.dinv = r.dinv;
  a.y = r.y;
  a.partials = r.red ? r.red->partials : nullptr;
  a.ticket = r.red ? r.red->ticket : nullptr;
  a.red_out = r.red_out;
  a.red_stride = r.red_stride;
  const int grid = row_grid(A, op, ctx->num_sms, set);
  const bool needs_red = (op == RowOp::SpmvDot || op == RowOp::SweepDot || op == RowOp::ResidDot2);
  PSC_REQUIRE(!needs_red || (r.red && r.red_out && grid <= r.red->grid), PSC_ERR_STATE, "reduction site missing");
  switch (op) {
    case RowOp::Spmv: row_kernel<RowOp::Spmv><<<grid, kBlock, 0, s>>>(a); break;
    case RowOp::SpmvDot: row_kernel<RowOp::SpmvDot><<<grid, kBlock, 0, s>>>(a); break;
    case RowOp::Sweep: row_kernel<RowOp::Sweep><<<grid, kBlock, 0, s>>>(a); break;
    case RowOp::SweepDot: row_kernel<RowOp::SweepDot><<<grid, kBlock, 0, s>>>(a); break;
    case RowOp::Resid: row_kernel<RowOp::Resid><<<grid, kBlock, 0, s>>>(a); break;
    case RowOp::ResidDot2: row_kernel<RowOp::ResidDot2><<<grid, kBlock, 0, s>>>(a); break;
    case RowOp::PAdd: row_kernel<RowOp::PAdd><<<grid, kBlock, 0, s>>>(a); break;
  }
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// ------------------------------------------------------------ vector kernels
static int vec_grid(psc_ctx* ctx, int64_t n) {
  const int64_t need = (n + kBlock - 1) / kBlock;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)ctx->num_sms * 8));
}

__global__ void __launch_bounds__(kBlock) scale_kernel(int64_t n, const double* __restrict__ dinv,
                                                       const double* __restrict__ b, double* __restrict__ x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = dinv[i] * b[i];
}

void launch_scale(psc_ctx* ctx, int64_t n, const double* dinv, const double* b, double* x, cudaStream_t s) {
  scale_kernel<<<vec_grid(ctx, n), kBlock, 0, s>>>(n, dinv, b, x);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// l1 diagonal from the sliced ELL: the diagonal entry is the first stored entry
// whose local column equals the local row (padding repeats the last column with
// value 0 and is skipped by the `found` flag); off-diagonal |a_ij| summed in
// stored order, then m = a_ii + sum.
__global__ void __launch_bounds__(kBlock) l1_dinv_kernel(const int64_t* __restrict__ sptr,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val, int64_t n,
                                                         double* __restrict__ dinv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i >> 5;
    const int lane = (int)(i & 31);
    const int64_t b = sptr[s];
    const int w = (int)((sptr[s + 1] - b) >> 5);
    double aii = 0.0, off = 0.0;
    bool found = false;
    for (int k = 0; k < w; ++k) {
      const int32_t c = col[b + 32 * k + lane];
      const double v = val[b + 32 * k + lane];
      if (c == (int32_t)i && !found) {
        aii = v;
        found = true;
      } else {
        off += fabs(v);
      }
    }
    dinv[i] = 1.0 / (aii + off);
  }
}

void launch_l1_dinv(psc_ctx* ctx, const Sell& A, double* dinv, cudaStream_t s) {
  if (A.n_rows == 0) return;
  l1_dinv_kernel<<<vec_grid(ctx, A.n_rows), kBlock, 0, s>>>(A.slice_ptr, A.col, A.val, A.n_rows, dinv);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

__global__ void __launch_bounds__(kBlock) cg_update_kernel(int64_t n, double* __restrict__ x,
                                                           const double* __restrict__ p, double* __restrict__ r,
                                                           const double* __restrict__ q, const double* g_pq,
                                                           const double* rz_old, int nranks, double* partials,
                                                           unsigned int* ticket, double* out) {
  const double alpha = __ldcg(rz_old) / gsum(g_pq, nranks);
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = x[i] + alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    acc[0] += ri * ri;
  }
  grid_reduce<1>(acc, partials, ticket, out, 1);
}

void launch_cg_update(psc_ctx* ctx, int64_t n, double* x, const double* p, double* r, const double* q,
                      const double* g_pq, const double* rz_old, int nranks, const RedSite* red, double* red_out,
                      cudaStream_t s) {
  const int g = std::min(vec_grid(ctx, n), red->grid);
  cg_update_kernel<<<g, kBlock, 0, s>>>(n, x, p, r, q, g_pq, rz_old, nranks, red->partials, red->ticket, red_out);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

__global__ void __launch_bounds__(kBlock) xpby_kernel(int64_t n, const double* __restrict__ z, double* __restrict__ p,
                                                      const double* g_rz, double* rz_old, int nranks,
                                                      unsigned int* ticket) {
  const double rz = gsum(g_rz, nranks);
  const double beta = rz / __ldcg(rz_old);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
  // rz_old := rz once every CTA has read the old value
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int tk = atomicAdd(ticket, 1u);
    if (tk == gridDim.x - 1) {
      *rz_old = rz;
      *ticket = 0u;
    }
  }
}

void launch_xpby(psc_ctx* ctx, int64_t n, const double* z, double* p, const double* g_rz, double* rz_old, int nranks,
                 const RedSite* red, cudaStream_t s) {
  xpby_kernel<<<vec_grid(ctx, n), kBlock, 0, s>>>(n, z, p, g_rz, rz_old, nranks, red->ticket);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

__global__ void __launch_bounds__(kBlock) dot_kernel(int64_t n, const double* __restrict__ a,
                                                     const double* __restrict__ b, double* partials,
                                                     unsigned int* ticket, double* out) {
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc[0] += a[i] * b[i];
  grid_reduce<1>(acc, partials, ticket, out, 1);
}

void launch_dot(psc_ctx* ctx, int64_t n, const double* a, const double* b, const RedSite* red, double* red_out,
                cudaStream_t s) {
  const int g = std::min(vec_grid(ctx, n), red->grid);
  dot_kernel<<<g, kBlock, 0, s>>>(n, a, b, red->partials, red->ticket, red_out);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

__global__ void pack_kernel(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ x,
                            double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[idx[i]];
}

void launch_pack(psc_ctx* ctx, int64_t n, const int32_t* idx, const double* x, double* sendbuf, cudaStream_t s) {
  if (n == 0) return;
  pack_kernel<<<vec_grid(ctx, n), kBlock, 0, s>>>(n, idx, x, sendbuf);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

__global__ void gather_kernel(int64_t n, const int64_t* __restrict__ map, const double* __restrict__ in,
                              double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[map[i]];
}

void launch_gather(psc_ctx* ctx, int64_t n, const int64_t* map, const double* in, double* out, cudaStream_t s) {
  if (n == 0) return;
  gather_kernel<<<vec_grid(ctx, n), kBlock, 0, s>>>(n, map, in, out);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// ------------------------------------------------------------ coarsest solve
// One CTA runs the whole coarsest-level solver (l1-Jacobi "as coarse
// solver (30 iterations)"): the iterate lives in shared memory (double buffer),
// A_coarse and dinv come from L2.  Replaces 30 dependent launches by one.
constexpr int kCoarseThreads = 1024;
int64_t coarse_smem_rows() { return (200 * 1024) / (2 * sizeof(double)); }

__global__ void __launch_bounds__(kCoarseThreads) coarse_solve_kernel(const int64_t* __restrict__ sptr,
                                                                      const int32_t* __restrict__ col,
                                                                      const double* __restrict__ val, int64_t n,
                                                                      const double* __restrict__ dinv,
                                                                      const double* __restrict__ b,
                                                                      double* __restrict__ xout, int nsweeps) {
  extern __shared__ double sm[];
  double* xa = sm;
  double* xb = sm + n;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) xa[i] = (nsweeps > 0) ? dinv[i] * b[i] : 0.0;
  __syncthreads();
  for (int sw = 1; sw < nsweeps; ++sw) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const int64_t s = i >> 5;
      const int lane = (int)(i & 31);
      const int64_t bs = sptr[s];
      const int w = (int)((sptr[s + 1] - bs) >> 5);
      double sum = 0.0;
      for (int k = 0; k < w; ++k) sum = fma(val[bs + 32 * k + lane], xa[col[bs + 32 * k + lane]], sum);
      xb[i] = xa[i] + dinv[i] * (b[i] - sum);
    }
    __syncthreads();
    double* t = xa;
    xa = xb;
    xb = t;
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) xout[i] = xa[i];
}

void launch_coarse_solve(psc_ctx* ctx, const Sell& A, const double* dinv, const double* b, double* x, int nsweeps,
                         cudaStream_t s) {
  const int64_t n = A.n_rows;
  PSC_REQUIRE(n <= coarse_smem_rows(), PSC_ERR_STATE, "coarsest level too large for the one-CTA solver");
  PSC_REQUIRE(A.n_cols_local == n, PSC_ERR_STATE, "coarsest matrix must have no halo");
  const size_t smem = (size_t)std::max<int64_t>(n, 1) * 2 * sizeof(double);
  static bool attr = false;
  if (!attr) {
    PSC_CUDA(cudaFuncSetAttribute(coarse_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  coarse_solve_kernel<<<1, kCoarseThreads, smem, s>>>(A.slice_ptr, A.col, A.val, n, dinv, b, x, nsweeps);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// --------------------------------------------------------- CSR -> sliced ELL
__device__ __forceinline__ int32_t map_col(int64_t g, int64_t own_begin, int64_t n_own,
                                           const int64_t* __restrict__ halo, int64_t nh, int* err) {
  if (g >= own_begin && g < own_begin + n_own) return (int32_t)(g - own_begin);
  int64_t lo = 0, hi = nh;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (halo[mid] < g) lo = mid + 1;
    else hi = mid;
  }
  if (lo < nh && halo[lo] == g) return (int32_t)(n_own + lo);
  *err = 1;
  return 0;
}

// one warp per slice: slice width (max row length) and whether any column is off-rank
__global__ void sell_width_kernel(int64_t n_rows, int64_t n_slices, const int64_t* __restrict__ rowptr,
                                  const int64_t* __restrict__ colg, int64_t own_begin, int64_t n_own,
                                  int64_t* __restrict__ slots, int32_t* __restrict__ bflag) {
  const int lane = threadIdx.x & 31;
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_slices) return;
  const int64_t i = s * 32 + lane;
  int len = 0, off = 0;
  if (i < n_rows) {
    const int64_t b = rowptr[i], e = rowptr[i + 1];
    len = (int)(e - b);
    for (int64_t k = b; k < e; ++k) {
      const int64_t g = colg[k];
      off |= (g < own_begin || g >= own_begin + n_own);
    }
  }
  for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
  off = __any_sync(0xffffffffu, off);
  if (lane == 0) {
    slots[s] = (int64_t)len * 32;
    bflag[s] = off;
  }
}

// thread per row: scatter the row into its slice column-major, renumbering columns
__global__ void sell_fill_kernel(int64_t n_rows, int64_t n_slices, const int64_t* __restrict__ rowptr,
                                 const int64_t* __restrict__ colg, const double* __restrict__ valcsr,
                                 const int64_t* __restrict__ sptr, int64_t own_begin, int64_t n_own,
                                 const int64_t* __restrict__ halo, int64_t nh, int32_t* __restrict__ col,
                                 double* __restrict__ val, int* err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_slices * 32) return;
  const int64_t s = i >> 5;
  const int lane = (int)(i & 31);
  const int64_t base = sptr[s];
  const int w = (int)((sptr[s + 1] - base) >> 5);
  int64_t b = 0, e = 0;
  if (i < n_rows) {
    b = rowptr[i];
    e = rowptr[i + 1];
  }
  int32_t last = 0;
  for (int k = 0; k < w; ++k) {
    const int64_t o = base + 32 * (int64_t)k + lane;
    if (b + k < e) {
      last = map_col(colg[b + k], own_begin, n_own, halo, nh, err);
      col[o] = last;
      val[o] = valcsr[b + k];
    } else {
      col[o] = last;
      val[o] = 0.0;
    }
  }
}

void sell_from_csr(psc_ctx* ctx, int64_t n_rows, const int64_t* d_rowptr, const int64_t* d_colg, const double* d_val,
                   int64_t nnz, int64_t own_begin, int64_t n_own, const int64_t* d_halo, int64_t n_halo, Sell& S,
                   cudaStream_t s) {
  S.n_rows = n_rows;
  S.n_cols_local = n_own + n_halo;
  S.nnz = nnz;
  S.n_slices = (n_rows + 31) / 32;
  S.slice_ptr = dalloc<int64_t>(S.n_slices + 1);
  int32_t* d_flag = dalloc<int32_t>(S.n_slices);
  int64_t* d_slots = dalloc<int64_t>(S.n_slices + 1);
  int* d_err = dalloc<int>(1);
  PSC_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  PSC_CUDA(cudaMemsetAsync(d_slots, 0, sizeof(int64_t) * (S.n_slices + 1), s));
  if (S.n_slices > 0) {
    const int64_t threads = S.n_slices * 32;
    sell_width_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(n_rows, S.n_slices, d_rowptr, d_colg,
                                                                         own_begin, n_own, d_slots, d_flag);
    PSC_CUDA(cudaGetLastError());
  }
  // exclusive scan of slots -> slice_ptr (n_slices + 1 entries)
  size_t tmp_bytes = 0;
  PSC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_slots, S.slice_ptr, S.n_slices + 1, s));
  void* d_tmp = dalloc<char>(tmp_bytes);
  PSC_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_slots, S.slice_ptr, S.n_slices + 1, s));
  PSC_CUDA(cudaMemcpyAsync(&S.padded, S.slice_ptr + S.n_slices, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(d_tmp);
  dfree(d_slots);
  S.col = dalloc<int32_t>(S.padded);
  S.val = dalloc<double>(S.padded);
  if (S.n_slices > 0) {
    const int64_t threads = S.n_slices * 32;
    sell_fill_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(n_rows, S.n_slices, d_rowptr, d_colg, d_val,
                                                                        S.slice_ptr, own_begin, n_own, d_halo,
                                                                        n_halo, S.col, S.val, d_err);
    PSC_CUDA(cudaGetLastError());
  }
  int h_err = 0;
  PSC_CUDA(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  std::vector<int32_t> flag(S.n_slices);
  if (S.n_slices)
    PSC_CUDA(cudaMemcpyAsync(flag.data(), d_flag, sizeof(int32_t) * S.n_slices, cudaMemcpyDeviceToHost, s));
  std::vector<int64_t> sp(S.n_slices + 1);
  PSC_CUDA(cudaMemcpyAsync(sp.data(), S.slice_ptr, sizeof(int64_t) * (S.n_slices + 1), cudaMemcpyDeviceToHost, s));
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(d_err);
  dfree(d_flag);
  PSC_REQUIRE(h_err == 0, PSC_ERR_STATE, "column not in the owned block nor in the assembled halo");
  std::vector<int32_t> in, bd;
  for (int64_t k = 0; k < S.n_slices; ++k) {
    (flag[k] ? bd : in).push_back((int32_t)k);
    S.max_width = std::max<int>(S.max_width, (int)((sp[k + 1] - sp[k]) / 32));
  }
  S.n_interior = (int64_t)in.size();
  S.n_boundary = (int64_t)bd.size();
  S.interior = dalloc<int32_t>(in.size());
  S.boundary = dalloc<int32_t>(bd.size());
  if (!in.empty())
    PSC_CUDA(cudaMemcpyAsync(S.interior, in.data(), sizeof(int32_t) * in.size(), cudaMemcpyHostToDevice, s));
  if (!bd.empty())
    PSC_CUDA(cudaMemcpyAsync(S.boundary, bd.data(), sizeof(int32_t) * bd.size(), cudaMemcpyHostToDevice, s));
  PSC_CUDA(cudaStreamSynchronize(s));
}

void sell_free(Sell& S) {
  dfree(S.slice_ptr);
  dfree(S.col);
  dfree(S.val);
  dfree(S.interior);
  dfree(S.boundary);
  S = Sell();
}

RedSite red_alloc(int num_sms, int nred) {
  RedSite r;
  r.grid = num_sms * 8;
  r.partials = dalloc<double>((size_t)r.grid * nred);
  r.ticket = dalloc<unsigned int>(1);
  PSC_CUDA(cudaMemset(r.ticket, 0, sizeof(unsigned int)));
  return r;
}

void red_free(RedSite& r) {
  dfree(r.partials);
  dfree(r.ticket);
  r = RedSite();
}

}  // namespace psc
