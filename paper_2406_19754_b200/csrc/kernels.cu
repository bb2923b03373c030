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

// Partial row sum of lane `sub` of a G-lane group over a contiguous padded row
// [b, e): entries b + sub, b + sub + G, ...; 4 independent loads in flight.
template <int G>
__device__ __forceinline__ double rg_row_sum(const int32_t* __restrict__ col, const double* __restrict__ val,
                                             int64_t b, int64_t e, int sub, const double* __restrict__ x) {
  double sum = 0.0;
  int64_t k = b + sub;
  for (; k + 3 * G < e; k += 4 * G) {
    int ci[4];
    double vi[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      ci[j] = __ldcs(col + k + j * G);
      vi[j] = __ldcs(val + k + j * G);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) sum = fma(vi[j], __ldg(x + ci[j]), sum);
  }
  for (; k < e; k += G) sum = fma(__ldcs(val + k), __ldg(x + __ldcs(col + k)), sum);
  return sum;
}

struct RowKArgs {
  const int64_t* ptr;
  const int32_t* col;
  const double* val;
  const int32_t* list;  // nullptr: units 0..nlist-1
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
struct NRed {
  static constexpr int value =
      (OP == RowOp::SpmvDot || OP == RowOp::SweepDot) ? 1 : (OP == RowOp::ResidDot2 ? 2 : 0);
};

// Fused epilogue of row i with row sum `sum`.
template <RowOp OP>
__device__ __forceinline__ void epilogue(const RowKArgs& a, int64_t i, double sum, double* acc) {
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

// sliced ELL: one warp per slice, one thread per row
template <RowOp OP>
__device__ __forceinline__ void sell_body(const RowKArgs& a) {
  constexpr int NR = NRed<OP>::value;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * kWarpsPerBlock;
  double acc[NR > 0 ? NR : 1] = {};
  for (int64_t t = (int64_t)blockIdx.x * kWarpsPerBlock + warp; t < a.nlist; t += stride) {
    const int64_t s = a.list ? (int64_t)a.list[t] : t;
    const double sum = sell_row_sum(a.ptr, a.col, a.val, s, lane, a.x);
    const int64_t i = s * kSlice + lane;
    if (i < a.n_rows) epilogue<OP>(a, i, sum, acc);
  }
  if constexpr (NR > 0) grid_reduce<NR>(acc, a.partials, a.ticket, a.red_out, a.red_stride);
}

// row groups: one warp per unit of 32/G rows, G lanes per row, fixed shuffle tree
template <RowOp OP, int G>
__device__ __forceinline__ void rg_body(const RowKArgs& a) {
  constexpr int NR = NRed<OP>::value;
  constexpr int RU = 32 / G;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int sub = lane & (G - 1);
  const int grp = lane / G;
  const int64_t stride = (int64_t)gridDim.x * kWarpsPerBlock;
  double acc[NR > 0 ? NR : 1] = {};
  for (int64_t t = (int64_t)blockIdx.x * kWarpsPerBlock + warp; t < a.nlist; t += stride) {
    const int64_t u = a.list ? (int64_t)a.list[t] : t;
    const int64_t i = u * RU + grp;
    int64_t b = 0, e = 0;
    if (i < a.n_rows) {
      b = a.ptr[i];
      e = a.ptr[i + 1];
    }
    double sum = rg_row_sum<G>(a.col, a.val, b, e, sub, a.x);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o, G);
    if (sub == 0 && i < a.n_rows) epilogue<OP>(a, i, sum, acc);
  }
  if constexpr (NR > 0) grid_reduce<NR>(acc, a.partials, a.ticket, a.red_out, a.red_stride);
}

// One named kernel per (layout, epilogue): readable launch lists and ncu filters.
#define PSC_ROW_KERNELS(name, OP)                                                                         \
  __global__ void __launch_bounds__(kBlock) sell_##name(RowKArgs a) { sell_body<OP>(a); }               \
  template <int G>                                                                                        \
  __global__ void __launch_bounds__(kBlock) rg_##name(RowKArgs a) {                                      \
    rg_body<OP, G>(a);                                                                                    \
  }
PSC_ROW_KERNELS(spmv, RowOp::Spmv)
PSC_ROW_KERNELS(spmv_dot, RowOp::SpmvDot)
PSC_ROW_KERNELS(sweep, RowOp::Sweep)
PSC_ROW_KERNELS(sweep_dot, RowOp::SweepDot)
PSC_ROW_KERNELS(resid, RowOp::Resid)
PSC_ROW_KERNELS(resid_dot2, RowOp::ResidDot2)
PSC_ROW_KERNELS(padd, RowOp::PAdd)
#undef PSC_ROW_KERNELS

using RowKernel = void (*)(RowKArgs);

template <int G>
static RowKernel rg_kernel(RowOp op) {
  switch (op) {
    case RowOp::Spmv: return rg_spmv<G>;
    case RowOp::SpmvDot: return rg_spmv_dot<G>;
    case RowOp::Sweep: return rg_sweep<G>;
    case RowOp::SweepDot: return rg_sweep_dot<G>;
    case RowOp::Resid: return rg_resid<G>;
    case RowOp::ResidDot2: return rg_resid_dot2<G>;
    case RowOp::PAdd: return rg_padd<G>;
  }
  return nullptr;
}

static RowKernel kernel_of(RowOp op, int lanes) {
  switch (lanes) {
    case 4: return rg_kernel<4>(op);
    case 8: return rg_kernel<8>(op);
    case 16: return rg_kernel<16>(op);
    case 32: return rg_kernel<32>(op);
    default: break;
  }
  switch (op) {
    case RowOp::Spmv: return sell_spmv;
    case RowOp::SpmvDot: return sell_spmv_dot;
    case RowOp::Sweep: return sell_sweep;
    case RowOp::SweepDot: return sell_sweep_dot;
    case RowOp::Resid: return sell_resid;
    case RowOp::ResidDot2: return sell_resid_dot2;
    case RowOp::PAdd: return sell_padd;
  }
  return nullptr;
}

static int lanes_slot(int lanes) { return lanes == 1 ? 0 : (lanes == 4 ? 1 : (lanes == 8 ? 2 : (lanes == 16 ? 3 : 4))); }

static int occ_for(RowOp op, int lanes) {
  static int occ[5][8] = {{-1, -1, -1, -1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1, -1, -1, -1},
                          {-1, -1, -1, -1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1, -1, -1, -1},
                          {-1, -1, -1, -1, -1, -1, -1, -1}};
  int& o = occ[lanes_slot(lanes)][(int)op];
  if (o < 0) {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel_of(op, lanes), kBlock, 0) != cudaSuccess || v < 1)
      v = 1;
    o = v;
  }
  return o;
}

static int64_t set_count(const Sell& A, SliceSet set) {
  return set == SliceSet::All ? A.n_units : (set == SliceSet::Interior ? A.n_interior : A.n_boundary);
}

int row_grid(const Sell& A, RowOp op, int num_sms, SliceSet set) {
  const int64_t n = set_count(A, set);
  const int64_t need = (n + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int64_t cap = (int64_t)num_sms * occ_for(op, A.lanes);
  return (int)std::max<int64_t>(1, std::min(need, cap));
}

void launch_rows(psc_ctx* ctx, const Sell& A, RowOp op, const RowArgs& r, cudaStream_t s, SliceSet set) {
  RowKArgs a;
  a.ptr = A.ptr;
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
  kernel_of(op, A.lanes)<<<grid, kBlock, 0, s>>>(a);
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

// l1 diagonal from either device layout: the diagonal entry is the
// first stored entry whose local column equals the local row (padding repeats
// the last column with value 0 and is skipped by the `found` flag);
// off-diagonal |a_ij| summed in stored order; m = a_ii + sum; dinv = 1/m.
__global__ void __launch_bounds__(kBlock) l1_dinv_kernel(const int64_t* __restrict__ ptr,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val, int64_t n, int lanes,
                                                         double* __restrict__ dinv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t base, step;
    int w;
    if (lanes == 1) {
      const int64_t s = i >> 5;
      base = ptr[s] + (i & 31);
      w = (int)((ptr[s + 1] - ptr[s]) >> 5);
      step = 32;
    } else {
      base = ptr[i];
      w = (int)(ptr[i + 1] - base);
      step = 1;
    }
    double aii = 0.0, off = 0.0;
    bool found = false;
    for (int k = 0; k < w; ++k) {
      const int32_t c = col[base + step * k];
      const double v = val[base + step * k];
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
  l1_dinv_kernel<<<vec_grid(ctx, A.n_rows), kBlock, 0, s>>>(A.ptr, A.col, A.val, A.n_rows, A.lanes, dinv);
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
// solver (30 iterations)"): iterate, right-hand side and dinv live in shared
// memory, A_coarse comes from L1/L2.  Replaces 30 dependent launches by one.
constexpr int kCoarseThreads = 1024;
constexpr int kCoarseSmem = 200 * 1024;
int64_t coarse_smem_rows() { return kCoarseSmem / (4 * sizeof(double)); }

struct CoarseArgs {
  const int64_t* ptr;
  const int32_t* col;
  const double* val;
  int64_t n;
  const double* dinv;
  const double* b;
  double* xout;
  int nsweeps;
};

// lanes == 1 (sliced ELL): one thread per row.  G > 1: G lanes per row.
template <int G>
__global__ void __launch_bounds__(kCoarseThreads) coarse_solve(CoarseArgs a) {
  extern __shared__ double sm[];
  const int64_t n = a.n;
  double* xa = sm;
  double* xb = sm + n;
  double* bs = sm + 2 * n;
  double* ds = sm + 3 * n;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    bs[i] = a.b[i];
    ds[i] = a.dinv[i];
    xa[i] = (a.nsweeps > 0) ? ds[i] * bs[i] : 0.0;  // first sweep from x = 0
  }
  __syncthreads();
  for (int sw = 1; sw < a.nsweeps; ++sw) {
    if constexpr (G == 1) {
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int64_t s = i >> 5;
        const int64_t base = a.ptr[s] + (i & 31);
        const int w = (int)((a.ptr[s + 1] - a.ptr[s]) >> 5);
        double sum = 0.0;
        for (int k = 0; k < w; ++k) sum = fma(__ldg(a.val + base + 32 * k), xa[__ldg(a.col + base + 32 * k)], sum);
        xb[i] = xa[i] + ds[i] * (bs[i] - sum);
      }
    } else {
      constexpr int RU = 32 / G;
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const int sub = lane & (G - 1), grp = lane / G;
      for (int64_t r0 = (int64_t)warp * RU; r0 < n; r0 += (int64_t)(kCoarseThreads / 32) * RU) {
        const int64_t i = r0 + grp;
        int64_t b = 0, e = 0;
        if (i < n) {
          b = a.ptr[i];
          e = a.ptr[i + 1];
        }
        double sum = 0.0;
        for (int64_t k = b + sub; k < e; k += G) sum = fma(__ldg(a.val + k), xa[__ldg(a.col + k)], sum);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o, G);
        if (sub == 0 && i < n) xb[i] = xa[i] + ds[i] * (bs[i] - sum);
      }
    }
    __syncthreads();
    double* t = xa;
    xa = xb;
    xb = t;
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a.xout[i] = xa[i];
}

template <int G>
static void coarse_launch(const CoarseArgs& a, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    PSC_CUDA(cudaFuncSetAttribute(coarse_solve<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCoarseSmem));
    attr = true;
  }
  const size_t smem = (size_t)std::max<int64_t>(a.n, 1) * 4 * sizeof(double);
  coarse_solve<G><<<1, kCoarseThreads, smem, s>>>(a);
}

void launch_coarse_solve(psc_ctx* ctx, const Sell& A, const double* dinv, const double* b, double* x, int nsweeps,
                         cudaStream_t s) {
  const int64_t n = A.n_rows;
  PSC_REQUIRE(n <= coarse_smem_rows(), PSC_ERR_STATE, "coarsest level too large for the one-CTA solver");
  PSC_REQUIRE(A.n_cols_local == n, PSC_ERR_STATE, "coarsest matrix must have no halo");
  CoarseArgs a{A.ptr, A.col, A.val, n, dinv, b, x, nsweeps};
  switch (A.lanes) {
    case 4: coarse_launch<4>(a, s); break;
    case 8: coarse_launch<8>(a, s); break;
    case 16: coarse_launch<16>(a, s); break;
    case 32: coarse_launch<32>(a, s); break;
    default: coarse_launch<1>(a, s); break;
  }
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

// row groups: padded row length (multiple of G) and off-rank flag per row
__global__ void rg_len_kernel(int64_t n_rows, int G, const int64_t* __restrict__ rowptr,
                              const int64_t* __restrict__ colg, int64_t own_begin, int64_t n_own,
                              int64_t* __restrict__ plen, int32_t* __restrict__ rflag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  const int64_t b = rowptr[i], e = rowptr[i + 1];
  int off = 0;
  for (int64_t k = b; k < e; ++k) {
    const int64_t g = colg[k];
    off |= (g < own_begin || g >= own_begin + n_own);
  }
  plen[i] = ((e - b + G - 1) / G) * G;
  rflag[i] = off;
}

__global__ void rg_fill_kernel(int64_t n_rows, const int64_t* __restrict__ rowptr, const int64_t* __restrict__ colg,
                               const double* __restrict__ valcsr, const int64_t* __restrict__ ptr, int64_t own_begin,
                               int64_t n_own, const int64_t* __restrict__ halo, int64_t nh, int32_t* __restrict__ col,
                               double* __restrict__ val, int* err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  const int64_t b = rowptr[i], e = rowptr[i + 1];
  const int64_t o0 = ptr[i], o1 = ptr[i + 1];
  int32_t last = 0;
  for (int64_t k = 0; k < o1 - o0; ++k) {
    if (b + k < e) {
      last = map_col(colg[b + k], own_begin, n_own, halo, nh, err);
      col[o0 + k] = last;
      val[o0 + k] = valcsr[b + k];
    } else {
      col[o0 + k] = last;
      val[o0 + k] = 0.0;
    }
  }
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// Layout choice: short rows (mean < PSC_RG_MIN = 10) -> sliced ELL,
// thread per row; long rows -> G lanes per row, G = pow2floor(mean / PSC_RG_DIV)
// clamped to [4, 32].  PSC_LANES forces a layout (1, 4, 8, 16, 32).
int choose_lanes(int64_t n_rows, int64_t nnz) {
  const int forced = env_int("PSC_LANES", 0);
  if (forced == 1 || forced == 4 || forced == 8 || forced == 16 || forced == 32) return forced;
  const double mu = n_rows ? (double)nnz / (double)n_rows : 0.0;
  if (mu < env_int("PSC_RG_MIN", 10)) return 1;
  const double t = mu / std::max(1, env_int("PSC_RG_DIV", 4));
  int G = 4;
  while (G * 2 <= t && G < 32) G *= 2;
  return G;
}

void sell_from_csr(psc_ctx* ctx, int64_t n_rows, const int64_t* d_rowptr, const int64_t* d_colg, const double* d_val,
                   int64_t nnz, int64_t own_begin, int64_t n_own, const int64_t* d_halo, int64_t n_halo, Sell& S,
                   cudaStream_t s, int lanes) {
  S.n_rows = n_rows;
  S.n_cols_local = n_own + n_halo;
  S.nnz = nnz;
  S.lanes = lanes > 0 ? lanes : choose_lanes(n_rows, nnz);
  const int RU = S.rows_per_unit();
  S.n_units = (n_rows + RU - 1) / RU;
  const bool sell = (S.lanes == 1);
  const int64_t nptr = sell ? S.n_units + 1 : n_rows + 1;
  S.ptr = dalloc<int64_t>(nptr);
  int32_t* d_flag = dalloc<int32_t>(sell ? S.n_units : n_rows);
  int64_t* d_len = dalloc<int64_t>(nptr);
  int* d_err = dalloc<int>(1);
  PSC_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  PSC_CUDA(cudaMemsetAsync(d_len, 0, sizeof(int64_t) * nptr, s));
  if (sell && S.n_units > 0) {
    const int64_t threads = S.n_units * 32;
    sell_width_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(n_rows, S.n_units, d_rowptr, d_colg,
                                                                         own_begin, n_own, d_len, d_flag);
    PSC_CUDA(cudaGetLastError());
  } else if (!sell && n_rows > 0) {
    rg_len_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, s>>>(n_rows, S.lanes, d_rowptr, d_colg, own_begin,
                                                                    n_own, d_len, d_flag);
    PSC_CUDA(cudaGetLastError());
  }
  size_t tmp_bytes = 0;
  PSC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_len, S.ptr, nptr, s));
  void* d_tmp = dalloc<char>(tmp_bytes);
  PSC_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_len, S.ptr, nptr, s));
  PSC_CUDA(cudaMemcpyAsync(&S.padded, S.ptr + nptr - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(d_tmp);
  dfree(d_len);
  S.col = dalloc<int32_t>(S.padded);
  S.val = dalloc<double>(S.padded);
  if (sell && S.n_units > 0) {
    const int64_t threads = S.n_units * 32;
    sell_fill_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(n_rows, S.n_units, d_rowptr, d_colg, d_val,
                                                                        S.ptr, own_begin, n_own, d_halo, n_halo,
                                                                        S.col, S.val, d_err);
    PSC_CUDA(cudaGetLastError());
  } else if (!sell && n_rows > 0) {
    rg_fill_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, s>>>(n_rows, d_rowptr, d_colg, d_val, S.ptr,
                                                                     own_begin, n_own, d_halo, n_halo, S.col, S.val,
                                                                     d_err);
    PSC_CUDA(cudaGetLastError());
  }
  int h_err = 0;
  PSC_CUDA(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  const int64_t nflag = sell ? S.n_units : n_rows;
  std::vector<int32_t> flag(nflag);
  if (nflag) PSC_CUDA(cudaMemcpyAsync(flag.data(), d_flag, sizeof(int32_t) * nflag, cudaMemcpyDeviceToHost, s));
  std::vector<int64_t> hp(nptr);
  PSC_CUDA(cudaMemcpyAsync(hp.data(), S.ptr, sizeof(int64_t) * nptr, cudaMemcpyDeviceToHost, s));
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(d_err);
  dfree(d_flag);
  PSC_REQUIRE(h_err == 0, PSC_ERR_STATE, "column not in the owned block nor in the assembled halo");
  std::vector<int32_t> in, bd;
  for (int64_t u = 0; u < S.n_units; ++u) {
    int f = 0;
    if (sell) {
      f = flag[u];
      S.max_width = std::max<int>(S.max_width, (int)((hp[u + 1] - hp[u]) / 32));
    } else {
      for (int64_t i = u * RU; i < std::min<int64_t>(n_rows, (u + 1) * RU); ++i) {
        f |= flag[i];
        S.max_width = std::max<int>(S.max_width, (int)(hp[i + 1] - hp[i]));
      }
    }
    (f ? bd : in).push_back((int32_t)u);
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
  dfree(S.ptr);
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
