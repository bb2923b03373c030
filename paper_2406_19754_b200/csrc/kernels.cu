// kernels.cu — sm_100a kernels of the AMG-PCG solve path (FP64, CUDA cores).
//
// Nothing on this path is a dense contraction ("arithmetic intensity is
// of order O(1) ... memory/communication-bound"), so there are no tensor-core
// ops: every kernel is written for HBM bandwidth — coalesced 8-byte per-lane
// streams of the sliced-ELL values/columns (evict-first, __ldcs), read-only
// cached gathers of x (__ldg, kept in the 126 MB L2), grid-stride loops sized
// to the SM count, and deterministic fixed-order reductions.
#include <algorithm>
#include <cub/cub.cuh>
#include <deque>
#include <numeric>

#include "kernels.h"

namespace psc {

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

template <typename... KArgs, typename... Args>
static void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  PSC_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// plain sliced-ELL kernels: minimum resident CTAs per SM requested from ptxas
// (2: ~116 registers; 3: 80; 4: 64 with spills: 3550 / 3523 / 3262 Mdof*it/s)
#ifndef PSC_SELL_MINB
#define PSC_SELL_MINB 2
#endif

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

constexpr int kHdr = 16;     // int32 words per slice header
constexpr int kMaxDiaHdr = 8;  // DIA offsets also held in the slice header (words 6..13)
constexpr int kMaxDia = 64;    // most diagonals a DIA slice may have (all in its column region)
// kEll16: ELL slice whose columns span less than 2^16 (all owned): stored as uint16
// offsets from a per-slice base column (header word 6), 2 bytes per slot instead of 4
enum SliceKind : int { kEll = 0, kDia = 1, kEll16 = 2 };

__device__ __forceinline__ int32_t load_hdr(const int32_t* __restrict__ hdr, int64_t s, int lane) {
  return lane < kHdr ? __ldg(hdr + s * kHdr + lane) : 0;
}

// DIA slice of width W (compile-time, so no predicates: all W value loads,
// then all W gathers, are in flight before the first FMA).  Column of entry j
// = i + offset_j (offsets broadcast from the header); an entry outside
// [0, ncols) is absent: its value is 0 and it gathers x[0] (a valid address),
// so fma(0, x[0], s) = s for finite x.
// matrix-stream load: evict-first unless the matrix is small enough to stay in L2
__device__ __forceinline__ double ldm(const double* p, bool keep) { return keep ? __ldg(p) : __ldcs(p); }
__device__ __forceinline__ int32_t ldm(const int32_t* p, bool keep) { return keep ? __ldg(p) : __ldcs(p); }
__device__ __forceinline__ int32_t ldm(const uint16_t* p, bool keep) {
  return (int32_t)(keep ? __ldg(reinterpret_cast<const unsigned short*>(p))
                        : __ldcs(reinterpret_cast<const unsigned short*>(p)));
}

// x gathers: read-only texture path, or (CG) through L2 only
template <bool CG>
__device__ __forceinline__ double ldx(const double* p) {
  if constexpr (CG) return __ldcg(p);
  else return __ldg(p);
}

template <int W, bool CG = false>
__device__ __forceinline__ double dia_sum(int32_t h, uint32_t i, const double* __restrict__ v,
                                          const double* __restrict__ x, uint32_t nc, bool keep) {
  double vi[W];
#pragma unroll
  for (int j = 0; j < W; ++j) vi[j] = ldm(v + 32 * j, keep);
  double xv[W];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    const uint32_t c = i + (uint32_t)__shfl_sync(0xffffffffu, h, 6 + j);
    xv[j] = ldx<CG>(x + (c < nc ? c : 0u));
  }
  double sum = 0.0;
#pragma unroll
  for (int j = 0; j < W; ++j) sum = fma(vi[j], xv[j], sum);
  return sum;
}

// ELL part of a row sum: columns c[32 k] (+ base: kEll16 offsets), batches of 8
// (value, column) loads issued before the dependent gathers
template <bool CG, typename CT>
__device__ __forceinline__ double ell_sum(const CT* __restrict__ c, int32_t base, int w, const double* __restrict__ v,
                                          const double* __restrict__ x, int64_t ncols, bool keep) {
  double sum = 0.0;
  int k = 0;
  for (; k + 8 <= w; k += 8) {
    int ci[8];
    double vi[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      ci[j] = base + ldm(c + 32 * j, keep);
      vi[j] = ldm(v + 32 * j, keep);
      PSC_DASSERT((uint64_t)ci[j] < (uint64_t)ncols);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) sum = fma(vi[j], ldx<CG>(x + ci[j]), sum);
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
        ci[j] = base + ldm(c + 32 * j, keep);
        vi[j] = ldm(v + 32 * j, keep);
      }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < rem) sum = fma(vi[j], ldx<CG>(x + ci[j]), sum);
  }
  return sum;
}

// Row sum of `lane`'s row i = 32 s + lane of slice s whose header word `h` this
// lane holds: s = sum_k val[k] * x[col[k]], k in stored order (padding adds
// fma(0, x, s) = s).  DIA slices: dia_sum<W>.  ELL slices: explicit columns,
// batches of 8 (value, column) loads issued before the dependent gathers.
// E16: the matrix has kEll16 slices.  The thread-per-row kernels come in two
// instantiations: without the kEll16 branch (116 registers for sell_sweep; the branch
// alone raised it to 128 and slowed the level-1 sweep) and with it.
template <bool CG = false, bool E16 = true>
__device__ __forceinline__ double sell_row_sum(int32_t h, int64_t s, int lane, const int32_t* __restrict__ col,
                                               const double* __restrict__ val, const double* __restrict__ x,
                                               int64_t ncols, bool keep) {
  const int64_t vb = ((int64_t)(uint32_t)__shfl_sync(0xffffffffu, h, 1) << 32) |
                     (uint32_t)__shfl_sync(0xffffffffu, h, 0);
  const int w = __shfl_sync(0xffffffffu, h, 4);
  const bool dia = __shfl_sync(0xffffffffu, h, 5) == 1;
  const double* v = val + vb + lane;
  if (dia) {
    // local indices < 2^31: unsigned 32-bit wrap-around maps out-of-range columns above ncols
    const uint32_t i = (uint32_t)(s * 32 + lane);
    const uint32_t nc = (uint32_t)ncols;
    switch (w) {
      case 1: return dia_sum<1, CG>(h, i, v, x, nc, keep);
      case 2: return dia_sum<2, CG>(h, i, v, x, nc, keep);
      case 3: return dia_sum<3, CG>(h, i, v, x, nc, keep);
      case 4: return dia_sum<4, CG>(h, i, v, x, nc, keep);
      case 5: return dia_sum<5, CG>(h, i, v, x, nc, keep);
      case 6: return dia_sum<6, CG>(h, i, v, x, nc, keep);
      case 7: return dia_sum<7, CG>(h, i, v, x, nc, keep);
      case 8: return dia_sum<8, CG>(h, i, v, x, nc, keep);
      default: break;
    }
    // wide DIA slice (level-1 Galerkin operators): the offsets, shared by the warp,
    // from the slice's column region (broadcast loads); the 32 lanes gather 32
    // consecutive entries of x per diagonal (coalesced, unlike ELL's scattered columns)
    const int64_t cbd = ((int64_t)(uint32_t)__shfl_sync(0xffffffffu, h, 3) << 32) |
                        (uint32_t)__shfl_sync(0xffffffffu, h, 2);
    const int32_t* offs = col + cbd;
    double sum = 0.0;
    int k = 0;
    for (; k + 8 <= w; k += 8) {
      double vi[8], xv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) vi[j] = ldm(v + 32 * (k + j), keep);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t c = i + (uint32_t)__ldg(offs + k + j);
        xv[j] = ldx<CG>(x + (c < nc ? c : 0u));
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) sum = fma(vi[j], xv[j], sum);
    }
    for (; k < w; ++k) {
      const uint32_t c = i + (uint32_t)__ldg(offs + k);
      sum = fma(ldm(v + 32 * k, keep), ldx<CG>(x + (c < nc ? c : 0u)), sum);
    }
    return sum;
  }
  const int64_t cb = ((int64_t)(uint32_t)__shfl_sync(0xffffffffu, h, 3) << 32) |
                     (uint32_t)__shfl_sync(0xffffffffu, h, 2);
  if constexpr (E16) {
    if (__shfl_sync(0xffffffffu, h, 5) == kEll16)
      return ell_sum<CG>(reinterpret_cast<const uint16_t*>(col + cb) + lane, __shfl_sync(0xffffffffu, h, 6), w, v,
                         x, ncols, keep);
  }
  return ell_sum<CG>(col + cb + lane, 0, w, v, x, ncols, keep);
}

// Column of entry k of local row i, stored in lane `lane` of slice s; -1 if a DIA
// offset points outside [0, ncols) (absent entry).
__device__ __forceinline__ int64_t sell_col(const int32_t* __restrict__ hdr, const int64_t* __restrict__ cptr,
                                            const int32_t* __restrict__ col, int64_t s, int lane, int64_t i, int k,
                                            int64_t ncols) {
  const int64_t cb = cptr[s];
  const int kind = hdr[s * kHdr + 5];
  if (kind == kDia) {
    const int64_t c = i + col[cb + k];
    return ((uint64_t)c < (uint64_t)ncols) ? c : -1;
  }
  if (kind == kEll16)
    return (int64_t)hdr[s * kHdr + 6] + reinterpret_cast<const uint16_t*>(col + cb)[32 * (int64_t)k + lane];
  return col[cb + 32 * (int64_t)k + lane];
}

// SELL-C-sigma (sigma = kSortWin = one 256-row TMA chunk): rows of a window are
// stored in slices in order of decreasing length.  perm[t] = row (offset in the
// window) held by slot t; iperm[i] = slot (offset in the window) of row i.  The
// row's entries, their order and its arithmetic are unchanged: only which lane
// computes it.  nullptr: identity.
constexpr int64_t kSortWin = 256;
__device__ __forceinline__ int64_t row_of_slot(const uint8_t* __restrict__ perm, int64_t t) {
  return perm ? (t & ~(kSortWin - 1)) + __ldg(perm + t) : t;
}
__device__ __forceinline__ int64_t slot_of_row(const uint8_t* __restrict__ iperm, int64_t i) {
  return iperm ? (i & ~(kSortWin - 1)) + __ldg(iperm + i) : i;
}

// Partial row sum of lane `sub` of a G-lane group over a contiguous padded row
// [b, e): entries b + sub, b + sub + G, ...; 4 independent loads in flight.
template <int G>
__device__ __forceinline__ double rg_row_sum(const int32_t* __restrict__ col, const double* __restrict__ val,
                                             int64_t b, int64_t e, int sub, const double* __restrict__ x,
                                             bool keep) {
  double sum = 0.0;
  int64_t k = b + sub;
  for (; k + 3 * G < e; k += 4 * G) {
    int ci[4];
    double vi[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      ci[j] = ldm(col + k + j * G, keep);
      vi[j] = ldm(val + k + j * G, keep);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) sum = fma(vi[j], __ldg(x + ci[j]), sum);
  }
  for (; k < e; k += G) sum = fma(ldm(val + k, keep), __ldg(x + ldm(col + k, keep)), sum);
  return sum;
}

struct RowKArgs {
  int keep_matrix;  // 1: matrix small enough to stay in L2 across the level's launches (evict_last)
  int xpre;         // square matrix, Spmv / PAdd: the TMA kernel bulk-copies the rows' own x block
                    // (evict_last) to bring the gathers' lines into L2 ahead of them
  const int64_t* ptr;
  const int64_t* cptr;
  const int32_t* hdr;
  int64_t ncols;
  const int32_t* col;
  const double* val;
  const uint8_t* perm;  // SELL-C-sigma slot -> row (nullptr: identity)
  const int32_t* list;  // nullptr: units 0..nlist-1
  int64_t nlist;
  int64_t n_rows;
  double alpha, beta;
  const double* x;
  const double* b;
  const double* dinv;
  double* y;
  double* y2;            // Spmv: if set, y2 = dinv2 .* y (first sweep from zero of the next level)
  const double* dinv2;
  const double* w;       // SweepDot: weight of the reduction (nullptr: b)
  double* partials;
  unsigned int* ticket;
  double* red_out;
  int red_stride;
  PushSpec push;
  WaitSpec wait;
};

template <RowOp OP>
struct NRed {
  static constexpr int value =
      (OP == RowOp::SpmvDot || OP == RowOp::SweepDot) ? 1 : (OP == RowOp::ResidDot2 ? 2 : 0);
};

// ------------------------------------------------------------ fused push
static __device__ __forceinline__ void fp_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
static __device__ __forceinline__ uint64_t fp_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// consumer: before any thread of the CTA reads x's halo, thread 0 waits until every
// neighbour's flag reached this rank's generation (the producer on each side signalled)
__device__ __forceinline__ void wait_halo(const WaitSpec& w) {
  if (threadIdx.x == 0) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    for (int q = 0; q < w.R; ++q)
      if (w.nbr[q]) {
        const uint64_t target = __ldcg(w.gen + q);
        while (fp_acquire_sys(w.myflag + q) < target) {
          uint64_t t;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
          if (t - t0 > w.timeout_ns) __trap();  // a peer that never signals: launch error, no hang
        }
      }
  }
  __syncthreads();
}
// producer epilogue: row i's new value into every neighbour slot it feeds
__device__ __forceinline__ void push_row(const PushSpec& p, int64_t i, double v) {
  if (!__ldg(p.sslice + (i >> 5))) return;  // most slices send nothing: one byte per 32 rows
  for (int t = __ldg(p.iptr + i); t < __ldg(p.iptr + i + 1); ++t) p.dst[__ldg(p.iq + t)][__ldg(p.ipos + t)] = v;
}
// producer end: the last CTA signals every neighbour once all CTAs' stores are visible
__device__ __forceinline__ void push_signal(const PushSpec& p) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    last = (atomicAdd(p.ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < p.R; ++q)
      if (p.nbr[q]) {
        const uint64_t g = p.gen[q] + 1;
        p.gen[q] = g;
        fp_release_sys(p.pflag[q], g);
      }
    *p.ticket = 0u;
  }
}

// Fused epilogue of row i with row sum `sum`, split in two: the row's vector
// operands are loaded by epi_load BEFORE the row sum (so they travel with the
// matrix values instead of costing one more memory round trip afterwards),
// epi_store combines and writes.
struct EpiIn {
  double b, d, x;
};

template <RowOp OP>
__device__ __forceinline__ EpiIn epi_load(const RowKArgs& a, int64_t i) {
  EpiIn e{0.0, 0.0, 0.0};
  if constexpr (OP == RowOp::Spmv) {
    if (a.beta != 0.0) e.x = a.y[i];
    if (a.y2) e.d = __ldcs(a.dinv2 + i);  // before the row sum: off the critical path
  } else if constexpr (OP == RowOp::SpmvDot) {
    e.x = __ldg(a.x + i);
  } else if constexpr (OP == RowOp::Sweep || OP == RowOp::SweepDot) {
    e.b = __ldcs(a.b + i);
    e.d = __ldcs(a.dinv + i);
    e.x = __ldg(a.x + i);
  } else if constexpr (OP == RowOp::Resid || OP == RowOp::ResidDot2) {
    e.b = __ldcs(a.b + i);
  } else if constexpr (OP == RowOp::PAdd) {
    e.x = a.y[i];
  }
  return e;
}

template <RowOp OP>
__device__ __forceinline__ void epi_store(const RowKArgs& a, int64_t i, double sum, const EpiIn& e, double* acc) {
  if constexpr (OP == RowOp::Spmv) {
    const double v = (a.beta == 0.0) ? a.alpha * sum : a.alpha * sum + a.beta * e.x;
    a.y[i] = v;
    if (a.push.on) push_row(a.push, i, v);
    if (a.y2) a.y2[i] = e.d * v;
  } else if constexpr (OP == RowOp::SpmvDot) {
    a.y[i] = sum;
    acc[0] += e.x * sum;
  } else if constexpr (OP == RowOp::Sweep || OP == RowOp::SweepDot || OP == RowOp::Sweep0) {
    const double xn = e.x + e.d * (e.b - sum);
    a.y[i] = xn;
    if (a.push.on) push_row(a.push, i, xn);
    if constexpr (OP == RowOp::SweepDot) acc[0] += (a.w ? __ldg(a.w + i) : e.b) * xn;
  } else if constexpr (OP == RowOp::Resid) {
    a.y[i] = e.b - sum;
    if (a.push.on) push_row(a.push, i, e.b - sum);
  } else if constexpr (OP == RowOp::ResidDot2) {
    const double r = e.b - sum;
    a.y[i] = r;
    acc[0] += r * r;
    acc[1] += e.b * e.b;
  } else if constexpr (OP == RowOp::PAdd) {
    a.y[i] = e.x + sum;
    if (a.push.on) push_row(a.push, i, e.x + sum);
  }
}

template <RowOp OP>
__device__ __forceinline__ void epilogue(const RowKArgs& a, int64_t i, double sum, double* acc) {
  epi_store<OP>(a, i, sum, epi_load<OP>(a, i), acc);
}

// sliced ELL: one warp per slice, one thread per row; the next slice's header
// is loaded before the current slice is processed (one dependent round trip
// less per slice)
template <RowOp OP, bool E16>
__device__ __forceinline__ void sell_body(const RowKArgs& a) {
  if (a.wait.on) wait_halo(a.wait);
  constexpr int NR = NRed<OP>::value;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * kWarpsPerBlock;
  double acc[NR > 0 ? NR : 1] = {};
  int64_t t = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
  int64_t s = 0;
  int32_t h = 0;
  if (t < a.nlist) {
    s = a.list ? (int64_t)a.list[t] : t;
    h = load_hdr(a.hdr, s, lane);
  }
  while (t < a.nlist) {
    const int64_t tn = t + stride;
    int64_t sn = 0;
    int32_t hn = 0;
    if (tn < a.nlist) {
      sn = a.list ? (int64_t)a.list[tn] : tn;
      hn = load_hdr(a.hdr, sn, lane);
    }
    const int64_t i = row_of_slot(a.perm, s * kSlice + lane);
    const bool live = i < a.n_rows;
    EpiIn e{0.0, 0.0, 0.0};
    if (live) e = epi_load<OP>(a, i);
    const double sum = sell_row_sum<false, E16>(h, s, lane, a.col, a.val, a.x, a.ncols, a.keep_matrix != 0);
    if (live) epi_store<OP>(a, i, sum, e, acc);
    t = tn;
    s = sn;
    h = hn;
  }
  if (a.push.on) push_signal(a.push);
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
    double sum = rg_row_sum<G>(a.col, a.val, b, e, sub, a.x, a.keep_matrix != 0);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o, G);
    if (sub == 0 && i < a.n_rows) epilogue<OP>(a, i, sum, acc);
  }
  if constexpr (NR > 0) grid_reduce<NR>(acc, a.partials, a.ticket, a.red_out, a.red_stride);
}

// One named kernel per (layout, epilogue): readable launch lists and ncu filters.
#define PSC_ROW_KERNELS(name, OP)                                                                         \
  __global__ void __launch_bounds__(kBlock, PSC_SELL_MINB) sell_##name(RowKArgs a) {                    \
    sell_body<OP, false>(a);                                                                              \
  }                                                                                                       \
  __global__ void __launch_bounds__(kBlock, PSC_SELL_MINB) sell16_##name(RowKArgs a) {                  \
    sell_body<OP, true>(a);                                                                               \
  }                                                                                                       \
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
    case RowOp::Sweep0: break;
  }
  return nullptr;
}

static RowKernel kernel_of(RowOp op, int lanes, bool e16 = false) {
  if (lanes == 1 && e16) {
    switch (op) {
      case RowOp::Spmv: return sell16_spmv;
      case RowOp::SpmvDot: return sell16_spmv_dot;
      case RowOp::Sweep: return sell16_sweep;
      case RowOp::SweepDot: return sell16_sweep_dot;
      case RowOp::Resid: return sell16_resid;
      case RowOp::ResidDot2: return sell16_resid_dot2;
      case RowOp::PAdd: return sell16_padd;
      case RowOp::Sweep0: break;
    }
    return nullptr;
  }
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
    case RowOp::Sweep0: break;
  }
  return nullptr;
}

static int lanes_slot(int lanes) { return lanes == 1 ? 0 : (lanes == 4 ? 1 : (lanes == 8 ? 2 : (lanes == 16 ? 3 : 4))); }

static int occ_for(RowOp op, int lanes, bool e16 = false) {
  static int occ[6][8] = {{-1, -1, -1, -1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1, -1, -1, -1},
                          {-1, -1, -1, -1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1, -1, -1, -1},
                          {-1, -1, -1, -1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1, -1, -1, -1}};
  const bool e = e16 && lanes == 1;
  int& o = occ[e ? 5 : lanes_slot(lanes)][(int)op];
  if (o < 0) {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel_of(op, lanes, e), kBlock, 0) != cudaSuccess || v < 1)
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
  const int64_t cap = (int64_t)num_sms * occ_for(op, A.lanes, A.n_e16 > 0);
  return (int)std::max<int64_t>(1, std::min(need, cap));
}

// ------------------------------------------------ TMA-staged sliced-ELL kernel
// Persistent CTAs, warp-specialised: warp 8 (one elected lane) streams chunks of
// 8 slices (256 rows) into a 3-stage shared-memory ring with 1-D bulk TMA copies
// (cp.async.bulk ... mbarrier::complete_tx): slice headers, values, explicit
// columns and the rows' epilogue vectors (b, dinv, own x / y), tracked by
// `full` mbarriers (expected transaction bytes).  Warps 0-7 each take one
// slice of the chunk: values and columns from shared memory, gathers of x
// from L2, fused epilogue, then arrive on the stage's `empty` mbarrier.  The
// bytes in flight per SM are set by the ring (2 CTAs x 3 stages x ~30 KB), not
// by registers or compiler scheduling.
constexpr int kTmaSlices = 8;                 // slices per chunk (= consumer warps)
constexpr int kTmaMaxW = 8;                   // widest slice the ring holds
constexpr int kTmaStages = 3;
constexpr int kTmaThreads = (kTmaSlices + 1) * 32;
constexpr int kTmaRows = kTmaSlices * 32;
static_assert(kTmaRows == kSortWin, "a TMA chunk must be one SELL-C-sigma sorting window");
constexpr int kTmaHdrBytes = kTmaSlices * kHdr * 4;                    // 512
constexpr int kTmaValBytes = kTmaSlices * kTmaMaxW * 32 * 8;           // 16 KB
constexpr int kTmaColBytes = kTmaSlices * kTmaMaxW * 32 * 4;           // 8 KB
constexpr int kTmaVecBytes = kTmaRows * 8;                             // 2 KB per vector
// Ring layouts by the matrix's slice kinds.  kRingAny: 3 stages with an int32 column
// region.  kRingDia (every slice DIA with its offsets in the header: A_0 of a stencil):
// no column region, so the same shared memory holds 4 stages.  kRingE16 (every slice
// DIA or kEll16: P_0): a uint16 column region, 4 stages.  More bytes in flight per SM:
// level-0 sweep 229.6 -> 224.8 us, Sweep0 259 -> 235, q = A p 217 -> 202 (same box).
enum TmaRingKind : int { kRingAny = 0, kRingDia = 1, kRingE16 = 2, kRingDia33 = 3, kRingDia42 = 4, kRingE16x3 = 5,
                         kRingAny3 = 6 };
template <int RING>
struct TmaRing {
  // kRingDia33 / kRingDia42: DIA-only rings for three CTAs per SM (3 stages each) or four
  // (2 stages each): more consumer warps per SM for the same bytes in flight
  static constexpr int kStages =
      RING == kRingAny ? kTmaStages
                       : (RING == kRingDia33 ? 3 : ((RING == kRingDia42 || RING == kRingE16x3 || RING == kRingAny3) ? 2 : 4));
  static constexpr int kColBytes =
      (RING == kRingAny || RING == kRingAny3) ? kTmaColBytes
                       : ((RING == kRingDia || RING == kRingDia33 || RING == kRingDia42) ? 0 : kTmaColBytes / 2);
  static constexpr int kStageBytes = kTmaHdrBytes + kTmaValBytes + kColBytes + 3 * kTmaVecBytes;
  static constexpr int kSmem = kStages * kStageBytes + 2 * kStages * 8;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <RowOp OP>
struct EpiVecs {  // which row vectors the epilogue reads: b, dinv, x(own), y
  static constexpr bool B = (OP == RowOp::Sweep || OP == RowOp::SweepDot || OP == RowOp::Resid ||
                             OP == RowOp::ResidDot2 || OP == RowOp::Sweep0);
  static constexpr bool D = (OP == RowOp::Sweep || OP == RowOp::SweepDot || OP == RowOp::Sweep0);
  // sell_tma reads the stored dinv (recomputing M_ii per row per sweep made the
  // kernel FP64-divide bound: 317 vs 221 us on A_0 of 256^3)
  static constexpr bool D_SELL = D;
  static constexpr bool X = (OP == RowOp::Sweep || OP == RowOp::SweepDot || OP == RowOp::SpmvDot);
  // residual: the rows' own x block is bulk-copied although the epilogue does not
  // read it, to bring the gathers' lines into L2 ahead of the consumers (no extra
  // DRAM bytes: the gathers read them anyway); 236 -> ~215 us on A_0 of 256^3
  static constexpr bool XPRE = (OP == RowOp::Resid || OP == RowOp::ResidDot2);
  static constexpr bool Y = (OP == RowOp::PAdd || OP == RowOp::Spmv);
};

template <RowOp OP, int RING>
__global__ void __launch_bounds__(kTmaThreads) sell_tma(RowKArgs a, int64_t nchunks, int64_t n_slices) {
  constexpr int NR = NRed<OP>::value;
  using EV = EpiVecs<OP>;
  using RG = TmaRing<RING>;
  constexpr bool DIAONLY = RING == kRingDia || RING == kRingDia33 || RING == kRingDia42;
  constexpr int kTmaStages = RG::kStages;
  constexpr int kTmaStageBytes = RG::kStageBytes;
  constexpr int kTmaColBytes = RG::kColBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTmaStages * kTmaStageBytes);
  uint64_t* empty = full + kTmaStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool readY = EV::Y && !(OP == RowOp::Spmv && a.beta == 0.0);
  // Spmv with y2 = dinv2 .* y (the next level's first sweep): dinv2 staged in slot 1
  const bool readD2 = OP == RowOp::Spmv && a.y2 != nullptr;
  // square Spmv / PAdd (AINV's Z^T and Z): own x block prefetched into slot 0 (unused)
  const bool xpre = (OP == RowOp::Spmv || OP == RowOp::PAdd) && a.xpre != 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kTmaStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kTmaSlices);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (a.wait.on) wait_halo(a.wait);
  double acc[NR > 0 ? NR : 1] = {};
  if (warp == kTmaSlices) {
    // ---------------- producer (one lane)
    if (lane == 0) {
      uint64_t pol_stream, pol_keep;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
      const uint64_t pol_mat = a.keep_matrix ? pol_keep : pol_stream;
      int64_t c = blockIdx.x;
      int64_t vb0 = 0, vb1 = 0, cb0 = 0, cb1 = 0;
      if (c < nchunks) {
        const int64_t s0 = c * kTmaSlices, s1 = min(s0 + kTmaSlices, n_slices);
        vb0 = a.ptr[s0]; vb1 = a.ptr[s1]; cb0 = a.cptr[s0]; cb1 = a.cptr[s1];
      }
      for (int64_t it = 0; c < nchunks; ++it, c += gridDim.x) {
        // prefetch the next chunk's offsets before blocking on the ring
        const int64_t cn = c + gridDim.x;
        int64_t nvb0 = 0, nvb1 = 0, ncb0 = 0, ncb1 = 0;
        if (cn < nchunks) {
          const int64_t s0 = cn * kTmaSlices, s1 = min(s0 + kTmaSlices, n_slices);
          nvb0 = a.ptr[s0]; nvb1 = a.ptr[s1]; ncb0 = a.cptr[s0]; ncb1 = a.cptr[s1];
        }
        const int st = (int)(it % kTmaStages);
        if (it >= kTmaStages) mbar_wait(&empty[st], (uint32_t)((it / kTmaStages - 1) & 1));
        unsigned char* base = smem + st * kTmaStageBytes;
        const int64_t s0 = c * kTmaSlices, s1 = min(s0 + kTmaSlices, n_slices);
        const int64_t r0 = s0 * 32, r1 = min(s1 * 32, a.n_rows);
        const uint32_t hb = (uint32_t)(s1 - s0) * kHdr * 4;
        const uint32_t vbytes = (uint32_t)(vb1 - vb0) * 8;
        const uint32_t cbytes = DIAONLY ? 0u : (uint32_t)(cb1 - cb0) * 4;  // DIA: offsets in the header
        const uint32_t rbytes = r1 > r0 ? (uint32_t)(((r1 - r0) * 8 + 15) & ~15) : 0u;
        const uint32_t nvec = (EV::B ? 1 : 0) + (EV::D_SELL ? 1 : 0) +
                              ((EV::X || EV::XPRE) ? 1 : 0) + (readY ? 1 : 0) + (readD2 ? 1 : 0) +
                              (xpre ? 1 : 0);
        PSC_DASSERT(vbytes <= (uint32_t)kTmaValBytes && cbytes <= (uint32_t)(DIAONLY ? 0 : kTmaColBytes) &&
                    rbytes <= (uint32_t)kTmaVecBytes && hb <= (uint32_t)kTmaHdrBytes);
        mbar_expect_tx(&full[st], hb + vbytes + cbytes + nvec * rbytes);
        bulk_g2s(base, a.hdr + s0 * kHdr, hb, &full[st], pol_keep);
        if (vbytes) bulk_g2s(base + kTmaHdrBytes, a.val + vb0, vbytes, &full[st], pol_mat);
        if (cbytes) bulk_g2s(base + kTmaHdrBytes + kTmaValBytes, a.col + cb0, cbytes, &full[st], pol_mat);
        unsigned char* vec = base + kTmaHdrBytes + kTmaValBytes + kTmaColBytes;
        if (rbytes) {
          // Sweep0 gathers b and 1/M of the neighbouring rows too (x1 = M^-1 b on the fly):
          // keep the chunk's b / 1/M in L2 for them instead of evicting them first
          constexpr bool kGatherBD = (OP == RowOp::Sweep0);
          if constexpr (EV::B) bulk_g2s(vec, a.b + r0, rbytes, &full[st], kGatherBD ? pol_keep : pol_stream);
          if constexpr (EV::D_SELL)
            bulk_g2s(vec + kTmaVecBytes, a.dinv + r0, rbytes, &full[st], kGatherBD ? pol_keep : pol_stream);
          if constexpr (EV::X || EV::XPRE) bulk_g2s(vec + 2 * kTmaVecBytes, a.x + r0, rbytes, &full[st], pol_keep);
          if (readY) bulk_g2s(vec + 2 * kTmaVecBytes, a.y + r0, rbytes, &full[st], pol_stream);
          if (readD2) bulk_g2s(vec + kTmaVecBytes, a.dinv2 + r0, rbytes, &full[st], pol_stream);
          if (xpre) bulk_g2s(vec, a.x + r0, rbytes, &full[st], pol_keep);
        }
        vb0 = nvb0; vb1 = nvb1; cb0 = ncb0; cb1 = ncb1;
      }
    }
  } else {
    // ---------------- consumers: warp `warp` takes slice s0 + warp of each chunk
    const uint32_t nc = (uint32_t)a.ncols;
    int64_t c = blockIdx.x;
    for (int64_t it = 0; c < nchunks; ++it, c += gridDim.x) {
      const int st = (int)(it % kTmaStages);
      mbar_wait(&full[st], (uint32_t)((it / kTmaStages) & 1));
      const unsigned char* base = smem + st * kTmaStageBytes;
      const int32_t* hs = reinterpret_cast<const int32_t*>(base);
      const double* vs = reinterpret_cast<const double*>(base + kTmaHdrBytes);
      const int32_t* cs = reinterpret_cast<const int32_t*>(base + kTmaHdrBytes + kTmaValBytes);
      const double* vec = reinterpret_cast<const double*>(base + kTmaHdrBytes + kTmaValBytes + kTmaColBytes);
      const int64_t s0 = c * kTmaSlices;
      const int64_t s = s0 + warp;
      if (s < n_slices) {
        const int32_t h = lane < kHdr ? hs[warp * kHdr + lane] : 0;
        const int32_t h0 = hs[0], h1 = hs[1], h2 = hs[2], h3 = hs[3];  // chunk's first slice: stage bases
        const int64_t vbase = ((int64_t)(uint32_t)h1 << 32) | (uint32_t)h0;
        const int64_t cbase = ((int64_t)(uint32_t)h3 << 32) | (uint32_t)h2;
        const int64_t vb = ((int64_t)(uint32_t)__shfl_sync(0xffffffffu, h, 1) << 32) |
                           (uint32_t)__shfl_sync(0xffffffffu, h, 0);
        const int w = __shfl_sync(0xffffffffu, h, 4);
        const int kind = __shfl_sync(0xffffffffu, h, 5);
        const bool dia = DIAONLY || kind == kDia;
        const double* v = vs + (vb - vbase) + lane;
        const uint32_t i = (uint32_t)(s * 32 + lane);
        // x_j; Sweep0: x1_j = dinv_j b_j, the first sweep from zero (a correctly
        // rounded product, as the stand-alone scale kernel stores it)
        auto gx = [&](uint32_t c) -> double {
          if constexpr (OP == RowOp::Sweep0) return __dmul_rn(__ldg(a.dinv + c), __ldg(a.b + c));
          else return __ldg(a.x + c);
        };
        double xv[kTmaMaxW];
        if (dia) {
#pragma unroll
          for (int j = 0; j < kTmaMaxW; ++j) {
            const uint32_t cj = i + (uint32_t)__shfl_sync(0xffffffffu, h, 6 + j);
            xv[j] = (j < w) ? gx(cj < nc ? cj : 0u) : 0.0;
          }
        } else {
          const int64_t cb = ((int64_t)(uint32_t)__shfl_sync(0xffffffffu, h, 3) << 32) |
                             (uint32_t)__shfl_sync(0xffffffffu, h, 2);
          if (RING == kRingE16 || kind == kEll16) {
            const uint16_t* cc = reinterpret_cast<const uint16_t*>(cs + (cb - cbase)) + lane;
            const uint32_t base = (uint32_t)__shfl_sync(0xffffffffu, h, 6);
#pragma unroll
            for (int j = 0; j < kTmaMaxW; ++j) PSC_DASSERT(j >= w || base + cc[32 * j] < nc);
#pragma unroll
            for (int j = 0; j < kTmaMaxW; ++j) xv[j] = (j < w) ? gx(base + cc[32 * j]) : 0.0;
          } else {
            const int32_t* cc = cs + (cb - cbase) + lane;
#pragma unroll
            for (int j = 0; j < kTmaMaxW; ++j) PSC_DASSERT(j >= w || (uint32_t)cc[32 * j] < nc);
#pragma unroll
            for (int j = 0; j < kTmaMaxW; ++j) xv[j] = (j < w) ? gx((uint32_t)cc[32 * j]) : 0.0;
          }
        }
        double sum = 0.0;
#pragma unroll
        for (int j = 0; j < kTmaMaxW; ++j)
          if (j < w) sum = fma(v[32 * j], xv[j], sum);
        // row of this lane (SELL-C-sigma: the chunk is the sorting window, so the
        // row is in the chunk's staged vectors)
        const int rl = a.perm ? (int)__ldg(a.perm + s * 32 + lane) : warp * 32 + lane;
        const int64_t row = c * kTmaRows + rl;
        if (row < a.n_rows) {
          EpiIn e{0.0, 0.0, 0.0};
          if constexpr (EV::B) e.b = vec[rl];
          if constexpr (EV::D) e.d = vec[kTmaRows + rl];
          if constexpr (EV::X) e.x = vec[2 * kTmaRows + rl];
          if (readY) e.x = vec[2 * kTmaRows + rl];
          if (readD2) e.d = vec[kTmaRows + rl];
          if constexpr (OP == RowOp::Sweep0) e.x = __dmul_rn(e.d, e.b);  // x1_i
          epi_store<OP>(a, row, sum, e, acc);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  if (a.push.on) push_signal(a.push);
  if constexpr (NR > 0) grid_reduce<NR>(acc, a.partials, a.ticket, a.red_out, a.red_stride);
}

template <RowOp OP, int RING>
static void tma_launch_t(const RowKArgs& a, int grid, int64_t nchunks, int64_t n_slices, cudaStream_t s) {
  static bool attr = false;
  constexpr int smem = TmaRing<RING>::kSmem;
  if (!attr) {
    PSC_CUDA(cudaFuncSetAttribute(sell_tma<OP, RING>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  launch_k(sell_tma<OP, RING>, grid, kTmaThreads, smem, s, a, nchunks, n_slices);
}
template <RowOp OP>
static void tma_launch(const RowKArgs& a, int grid, int64_t nchunks, int64_t n_slices, int ring, cudaStream_t s) {
  if (ring == kRingDia) tma_launch_t<OP, kRingDia>(a, grid, nchunks, n_slices, s);
  else if (ring == kRingDia33) tma_launch_t<OP, kRingDia33>(a, grid, nchunks, n_slices, s);
  else if (ring == kRingDia42) tma_launch_t<OP, kRingDia42>(a, grid, nchunks, n_slices, s);
  else if (ring == kRingE16x3) tma_launch_t<OP, kRingE16x3>(a, grid, nchunks, n_slices, s);
  else if (ring == kRingAny3) tma_launch_t<OP, kRingAny3>(a, grid, nchunks, n_slices, s);
  else if (ring == kRingE16) tma_launch_t<OP, kRingE16>(a, grid, nchunks, n_slices, s);
  else tma_launch_t<OP, kRingAny>(a, grid, nchunks, n_slices, s);
}

// ---------------------------------------------- TMA-staged row-group kernel
// Same producer / consumer ring as sell_tma for the row-group layout: a chunk
// is 8 units (8 x 32/G consecutive rows, contiguous in memory); the producer
// bulk-copies the chunk's row pointers, values, columns and epilogue vectors;
// consumer warp w reduces unit w's rows with G lanes each (values/columns from
// shared memory, gathers of x from L2).
constexpr int kRgCap = 4096;                       // entries per stage
constexpr int kRgMaxRows = kTmaSlices * 8;         // 8 units x at most 8 rows (G = 4)
constexpr int kRgValBytes = kRgCap * 8;
constexpr int kRgColBytes = kRgCap * 4;
constexpr int kRgPtrBytes = 1024;                  // (kRgMaxRows + 1) int64, rounded
constexpr int kRgVecBytes = kRgMaxRows * 8;
constexpr int kRgStages = 2;
constexpr int kRgStageBytes = kRgValBytes + kRgColBytes + kRgPtrBytes + 3 * kRgVecBytes;
constexpr int kRgSmem = kRgStages * kRgStageBytes + 2 * kRgStages * 8;

template <RowOp OP, int G>
__global__ void __launch_bounds__(kTmaThreads) rg_tma(RowKArgs a, int64_t nchunks) {
  constexpr int NR = NRed<OP>::value;
  constexpr int RU = 32 / G;
  constexpr int CR = kTmaSlices * RU;  // rows per chunk
  using EV = EpiVecs<OP>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRgStages * kRgStageBytes);
  uint64_t* empty = full + kRgStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool readD2 = OP == RowOp::Spmv && a.y2 != nullptr;  // y2 = dinv2 .* y: dinv2 in slot 1
  const bool readY = EV::Y && !(OP == RowOp::Spmv && a.beta == 0.0);
  if (threadIdx.x == 0) {
    for (int st = 0; st < kRgStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kTmaSlices);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc[NR > 0 ? NR : 1] = {};
  if (warp == kTmaSlices) {
    if (lane == 0) {
      uint64_t pol_stream, pol_keep;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
      const uint64_t pol_mat = a.keep_matrix ? pol_keep : pol_stream;
      int64_t c = blockIdx.x;
      int64_t e0 = 0, e1 = 0;
      if (c < nchunks) {
        e0 = a.ptr[c * CR];
        e1 = a.ptr[min((c + 1) * CR, a.n_rows)];
      }
      for (int64_t it = 0; c < nchunks; ++it, c += gridDim.x) {
        const int64_t cn = c + gridDim.x;
        int64_t ne0 = 0, ne1 = 0;
        if (cn < nchunks) {
          ne0 = a.ptr[cn * CR];
          ne1 = a.ptr[min((cn + 1) * CR, a.n_rows)];
        }
        const int st = (int)(it % kRgStages);
        if (it >= kRgStages) mbar_wait(&empty[st], (uint32_t)((it / kRgStages - 1) & 1));
        unsigned char* base = smem + st * kRgStageBytes;
        const int64_t r0 = c * CR, r1 = min(r0 + CR, a.n_rows);
        const uint32_t pbytes = (uint32_t)(((r1 - r0 + 1) * 8 + 15) & ~15);
        const uint32_t vbytes = (uint32_t)(e1 - e0) * 8;
        const uint32_t cbytes = (uint32_t)(e1 - e0) * 4;
        const uint32_t rbytes = (uint32_t)(((r1 - r0) * 8 + 15) & ~15);
        const uint32_t nvec = (EV::B ? 1 : 0) + (EV::D ? 1 : 0) + (EV::X ? 1 : 0) + (readY ? 1 : 0) + (readD2 ? 1 : 0);
        PSC_DASSERT(e1 - e0 <= kRgCap && pbytes <= (uint32_t)kRgPtrBytes && r1 - r0 <= kRgMaxRows);
        mbar_expect_tx(&full[st], pbytes + vbytes + cbytes + nvec * rbytes);
        bulk_g2s(base + kRgValBytes + kRgColBytes, a.ptr + r0, pbytes, &full[st], pol_keep);
        if (vbytes) {
          bulk_g2s(base, a.val + e0, vbytes, &full[st], pol_mat);
          bulk_g2s(base + kRgValBytes, a.col + e0, cbytes, &full[st], pol_mat);
        }
        unsigned char* vec = base + kRgValBytes + kRgColBytes + kRgPtrBytes;
        if constexpr (EV::B) bulk_g2s(vec, a.b + r0, rbytes, &full[st], pol_stream);
        if constexpr (EV::D) bulk_g2s(vec + kRgVecBytes, a.dinv + r0, rbytes, &full[st], pol_stream);
        if constexpr (EV::X) bulk_g2s(vec + 2 * kRgVecBytes, a.x + r0, rbytes, &full[st], pol_keep);
        if (readY) bulk_g2s(vec + 2 * kRgVecBytes, a.y + r0, rbytes, &full[st], pol_stream);
        if (readD2) bulk_g2s(vec + kRgVecBytes, a.dinv2 + r0, rbytes, &full[st], pol_stream);
        e0 = ne0;
        e1 = ne1;
      }
    }
  } else {
    const int sub = lane & (G - 1), grp = lane / G;
    int64_t c = blockIdx.x;
    for (int64_t it = 0; c < nchunks; ++it, c += gridDim.x) {
      const int st = (int)(it % kRgStages);
      mbar_wait(&full[st], (uint32_t)((it / kRgStages) & 1));
      const unsigned char* base = smem + st * kRgStageBytes;
      const double* vs = reinterpret_cast<const double*>(base);
      const int32_t* cs = reinterpret_cast<const int32_t*>(base + kRgValBytes);
      const int64_t* ps = reinterpret_cast<const int64_t*>(base + kRgValBytes + kRgColBytes);
      const double* vec = reinterpret_cast<const double*>(base + kRgValBytes + kRgColBytes + kRgPtrBytes);
      const int lr = warp * RU + grp;  // row within the chunk
      const int64_t i = c * CR + lr;
      const bool live = i < a.n_rows;
      int b = 0, e = 0;
      if (live) {
        const int64_t e0 = ps[0];
        b = (int)(ps[lr] - e0);
        e = (int)(ps[lr + 1] - e0);
      }
      double sum = 0.0;
      for (int kk = b + sub; kk < e; kk += 8 * G) {
        int cj[8];
        double vj[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = kk + j * G;
          const bool ok = k < e;
          cj[j] = ok ? cs[k] : 0;
          vj[j] = ok ? vs[k] : 0.0;
        }
        double xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) xv[j] = __ldg(a.x + cj[j]);
#pragma unroll
        for (int j = 0; j < 8; ++j) sum = fma(vj[j], xv[j], sum);
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o, G);
      if (sub == 0 && live) {
        EpiIn ein{0.0, 0.0, 0.0};
        if constexpr (EV::B) ein.b = vec[lr];
        if constexpr (EV::D) ein.d = vec[kRgMaxRows + lr];
        if constexpr (EV::X) ein.x = vec[2 * kRgMaxRows + lr];
        if (readY) ein.x = vec[2 * kRgMaxRows + lr];
        if (readD2) ein.d = vec[kRgMaxRows + lr];
        epi_store<OP>(a, i, sum, ein, acc);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  if constexpr (NR > 0) grid_reduce<NR>(acc, a.partials, a.ticket, a.red_out, a.red_stride);
}

template <RowOp OP, int G>
static void rg_tma_launch(const RowKArgs& a, int grid, int64_t nchunks, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    PSC_CUDA(cudaFuncSetAttribute(rg_tma<OP, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRgSmem));
    attr = true;
  }
  launch_k(rg_tma<OP, G>, grid, kTmaThreads, kRgSmem, s, a, nchunks);
}

template <int G>
static void rg_tma_dispatch(RowOp op, const RowKArgs& a, int grid, int64_t nchunks, cudaStream_t s) {
  switch (op) {
    case RowOp::Spmv: rg_tma_launch<RowOp::Spmv, G>(a, grid, nchunks, s); break;
    case RowOp::SpmvDot: rg_tma_launch<RowOp::SpmvDot, G>(a, grid, nchunks, s); break;
    case RowOp::Sweep: rg_tma_launch<RowOp::Sweep, G>(a, grid, nchunks, s); break;
    case RowOp::SweepDot: rg_tma_launch<RowOp::SweepDot, G>(a, grid, nchunks, s); break;
    case RowOp::Resid: rg_tma_launch<RowOp::Resid, G>(a, grid, nchunks, s); break;
    case RowOp::ResidDot2: rg_tma_launch<RowOp::ResidDot2, G>(a, grid, nchunks, s); break;
    case RowOp::PAdd: rg_tma_launch<RowOp::PAdd, G>(a, grid, nchunks, s); break;
    case RowOp::Sweep0: break;
  }
}

static bool rg_tma_ok(const Sell& A, const RowArgs& r, SliceSet set) {
  const int off = env_int("PSC_NO_TMA", 0) || env_int("PSC_NO_RG_TMA", 0);
  return !off && A.lanes > 1 && A.max_chunk <= kRgCap && set == SliceSet::All && r.vec_padded && A.n_units > 0;
}

// TMA path: sliced ELL, every slice at most kTmaMaxW wide, all slices, vectors
// padded (the bulk copies of the last chunk's rows round up to 16 bytes).
static bool tma_ok(const Sell& A, const RowArgs& r, SliceSet set) {
  const int off = env_int("PSC_NO_TMA", 0);
  return !off && A.lanes == 1 && A.max_width <= kTmaMaxW && set == SliceSet::All && r.vec_padded && A.hdr &&
         A.n_units > 0;
}

const char* kt_name(const std::string& n) {  // interned kernel label for KTrace
  static std::deque<std::string> names;
  for (const auto& x : names)
    if (x == n) return x.c_str();
  names.push_back(n);
  return names.back().c_str();
}

static const char* op_name(RowOp op) {
  switch (op) {
    case RowOp::Spmv: return "Spmv";
    case RowOp::SpmvDot: return "SpmvDot";
    case RowOp::Sweep: return "Sweep";
    case RowOp::SweepDot: return "SweepDot";
    case RowOp::Resid: return "Resid";
    case RowOp::ResidDot2: return "ResidDot2";
    case RowOp::PAdd: return "PAdd";
    case RowOp::Sweep0: return "Sweep0";
  }
  return "?";
}

// Bytes one launch must move: algorithmic = SURVEY.md §8(d)'s count,
// 12 B per stored nonzero + 8 B per vector element read or written once (x counted
// once over the column space); layout = the same vectors + the matrix as stored
// (8 B per value slot incl. padding, 4 B per column slot, slice headers, row order).
static void row_bytes(const Sell& A, RowOp op, const RowArgs& r, double& alg, double& lay) {
  const double n = (double)A.n_rows, nc = (double)A.n_cols_local;
  double vec = 8.0 * nc;  // x gathered (Sweep0: b, then dinv, as x1 = dinv .* b)
  switch (op) {
    case RowOp::Spmv: vec += 8.0 * n * (1 + (r.beta != 0.0) + (r.y2 ? 2 : 0)); break;
    case RowOp::SpmvDot: vec += 8.0 * n; break;
    case RowOp::Sweep: vec += 24.0 * n; break;
    case RowOp::SweepDot: vec += 8.0 * n * (3 + (r.w ? 1 : 0)); break;
    case RowOp::Resid: case RowOp::ResidDot2: vec += 16.0 * n; break;
    case RowOp::PAdd: vec += 16.0 * n; break;
    case RowOp::Sweep0: vec = 24.0 * n; break;
  }
  const double hdr = A.lanes == 1 ? 64.0 * (double)A.n_units + (A.perm ? 32.0 * (double)A.n_units : 0.0)
                                  : 8.0 * (n + 1);
  alg = 12.0 * (double)A.nnz + vec;
  lay = 8.0 * (double)A.padded + 4.0 * (double)A.col_slots + hdr + vec;
}

bool rows_can_push(const Sell& A, const RowArgs& r) {
  return A.lanes == 1 && !A.perm && (tma_ok(A, r, SliceSet::All) || A.hdr != nullptr);
}

void launch_rows(psc_ctx* ctx, const Sell& A, RowOp op, const RowArgs& r, cudaStream_t s, SliceSet set) {
  if (op == RowOp::Sweep0 && !tma_ok(A, r, set)) {
    // two launches: x = dinv .* b, then one sweep from x
    launch_scale(ctx, A.n_rows, r.dinv, r.b, const_cast<double*>(r.x), s);
    launch_rows(ctx, A, RowOp::Sweep, r, s, set);
    return;
  }
  double alg = 0.0, lay = 0.0;
  const char* kname = nullptr;
  if (ctx->kt.on) {
    row_bytes(A, op, r, alg, lay);
    const char* fam = tma_ok(A, r, set) ? "sell_tma" : (A.lanes == 1 ? "sell" : (rg_tma_ok(A, r, set) ? "rg_tma" : "rg"));
    kname = kt_name(std::string(fam) + "<" + op_name(op) + (A.lanes > 1 ? "," + std::to_string(A.lanes) : "") +
                    ">" + (A.perm ? " sorted" : "") + (set != SliceSet::All ? " subset" : ""));
  }
  KtScope kts(ctx, s, kname, alg, lay);
  RowKArgs a;
  // matrices up to 48 MB stay in L2 (evict_last) across the 8-10 launches of their level
  a.keep_matrix = (A.padded * 12 + A.n_rows * 8) <= ((int64_t)env_int("PSC_KEEP_MB", 96) << 20) ? 1 : 0;
  a.xpre = (A.n_rows == A.n_cols_local && (op == RowOp::Spmv || op == RowOp::PAdd) && !env_int("PSC_NO_XPRE", 0)) ? 1 : 0;
  a.perm = A.perm;
  a.ptr = A.ptr;
  a.cptr = A.cptr;
  a.hdr = A.hdr;
  a.ncols = A.n_cols_local;
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
  a.y2 = r.y2;
  a.dinv2 = r.dinv2;
  a.w = r.w;
  a.partials = r.red ? r.red->partials : nullptr;
  a.ticket = r.red ? r.red->ticket : nullptr;
  a.red_out = r.red_out;
  a.red_stride = r.red_stride;
  a.push = r.push;
  a.wait = r.wait;
  PSC_REQUIRE(!(r.push.on || r.wait.on) || (set == SliceSet::All && rows_can_push(A, r)), PSC_ERR_STATE,
              "fused push / wait on a row kernel without them");
  const bool needs_red = (op == RowOp::SpmvDot || op == RowOp::SweepDot || op == RowOp::ResidDot2);
  if (tma_ok(A, r, set)) {
    const int64_t nchunks = (A.n_units + kTmaSlices - 1) / kTmaSlices;
    // ring layout by slice kinds (DIA slices here have <= 8 offsets, in the header)
    int dia4 = kRingAny;
    if (!env_int("PSC_NO_TMA4", 0)) {
      if (A.n_dia == A.n_units) {
        // same-box A/B on A_0 of 256^3 (2x4 / 3x3 / 4x2 CTAs x stages): the sweeps and the
        // residual are fastest at 4x2 (222 / 201 us), Sweep0 (two gathers per entry) and
        // q = A p at 3x3 (236 / 192 us); PSC_TMA_RING=1|3|4 forces one layout
        const int e = env_int("PSC_TMA_RING", 0);
        if (e == 1) dia4 = kRingDia;
        else if (e == 3) dia4 = kRingDia33;
        else if (e == 4) dia4 = kRingDia42;
        else dia4 = (op == RowOp::Sweep0 || op == RowOp::SpmvDot) ? kRingDia33 : kRingDia42;
      }
      // DIA / 16-bit-column matrices (P_0): 3 CTAs x 2 stages (P_0 of 256^3: 191 vs 197.5 us
      // at 2 x 4); PSC_TMA_RING_E16=2 keeps 2 x 4
      else if (A.n_dia + A.n_e16 == A.n_units) dia4 = env_int("PSC_TMA_RING_E16", 3) == 2 ? kRingE16 : kRingE16x3;
    }
    // CTAs per SM the ring's shared memory allows
    // mixed slice kinds (a distributed A_0: its boundary slices reference halo columns, so
    // they are int32 ELL): 3 CTAs x 2 stages (2 B200: q = A p 216 -> 205 us, P_0 198 ->
    // 191, residual 218 -> 213; 7094 -> 7187 Mdof*iters/s); PSC_TMA_RING_ANY=2: 2 x 3
    if (dia4 == kRingAny && env_int("PSC_TMA_RING_ANY", 3) != 2) dia4 = kRingAny3;
    const int per_sm = (dia4 == kRingDia33 || dia4 == kRingE16x3 || dia4 == kRingAny3) ? 3 : (dia4 == kRingDia42 ? 4 : 2);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nchunks, per_sm * (int64_t)ctx->num_sms));
    PSC_REQUIRE(!needs_red || (r.red && r.red_out && grid <= r.red->grid), PSC_ERR_STATE, "reduction site missing");
    switch (op) {
      case RowOp::Spmv: tma_launch<RowOp::Spmv>(a, grid, nchunks, A.n_units, dia4, s); break;
      case RowOp::SpmvDot: tma_launch<RowOp::SpmvDot>(a, grid, nchunks, A.n_units, dia4, s); break;
      case RowOp::Sweep: tma_launch<RowOp::Sweep>(a, grid, nchunks, A.n_units, dia4, s); break;
      case RowOp::SweepDot: tma_launch<RowOp::SweepDot>(a, grid, nchunks, A.n_units, dia4, s); break;
      case RowOp::Resid: tma_launch<RowOp::Resid>(a, grid, nchunks, A.n_units, dia4, s); break;
      case RowOp::ResidDot2: tma_launch<RowOp::ResidDot2>(a, grid, nchunks, A.n_units, dia4, s); break;
      case RowOp::PAdd: tma_launch<RowOp::PAdd>(a, grid, nchunks, A.n_units, dia4, s); break;
      case RowOp::Sweep0: tma_launch<RowOp::Sweep0>(a, grid, nchunks, A.n_units, dia4, s); break;
    }
    PSC_CUDA(cudaGetLastError());
    ctx->launches++;
    return;
  }
  if (rg_tma_ok(A, r, set)) {
    const int64_t nchunks = (A.n_units + kTmaSlices - 1) / kTmaSlices;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nchunks, 2 * (int64_t)ctx->num_sms));
    PSC_REQUIRE(!needs_red || (r.red && r.red_out && grid <= r.red->grid), PSC_ERR_STATE, "reduction site missing");
    switch (A.lanes) {
      case 4: rg_tma_dispatch<4>(op, a, grid, nchunks, s); break;
      case 8: rg_tma_dispatch<8>(op, a, grid, nchunks, s); break;
      case 16: rg_tma_dispatch<16>(op, a, grid, nchunks, s); break;
      default: rg_tma_dispatch<32>(op, a, grid, nchunks, s); break;
    }
    PSC_CUDA(cudaGetLastError());
    ctx->launches++;
    return;
  }
  const int grid = row_grid(A, op, ctx->num_sms, set);
  PSC_REQUIRE(!needs_red || (r.red && r.red_out && grid <= r.red->grid), PSC_ERR_STATE, "reduction site missing");
  launch_k(kernel_of(op, A.lanes, A.n_e16 > 0), grid, kBlock, 0, s, a);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// ------------------------------------------------------------ vector kernels
static int vec_grid(psc_ctx* ctx, int64_t n) {
  const int64_t need = (n + kBlock - 1) / kBlock;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)ctx->num_sms * 8));
}

// Vector kernels: cg_update and fcg_dir move two elements per thread and
// iteration with 16-byte accesses (library buffers are 256-byte aligned; the odd
// tail element by thread 0).
__device__ __forceinline__ double2 ld2(const double* p, int64_t j) { return reinterpret_cast<const double2*>(p)[j]; }
__device__ __forceinline__ void st2(double* p, int64_t j, double2 v) { reinterpret_cast<double2*>(p)[j] = v; }

__global__ void __launch_bounds__(kBlock) scale_kernel(int64_t n, const double* __restrict__ dinv,
                                                       const double* __restrict__ b, double* __restrict__ x) {  // (16-byte form measured 57 vs 56 us: kept scalar)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = dinv[i] * b[i];
}

static bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

void launch_scale(psc_ctx* ctx, int64_t n, const double* dinv, const double* b, double* x, cudaStream_t s) {
  KtScope kts(ctx, s, "scale", 24.0 * n, 24.0 * n);
  PSC_REQUIRE(al16(dinv) && al16(b) && al16(x), PSC_ERR_STATE, "vector kernels need 16-byte aligned buffers");
  launch_k(scale_kernel, vec_grid(ctx, n), kBlock, 0, s, n, dinv, b, x);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// l1 diagonal from either device layout: the diagonal entry is the
// first stored entry whose local column equals the local row (padding repeats
// the last column with value 0 and is skipped by the `found` flag);
// off-diagonal |a_ij| summed in stored order; m = a_ii + sum; dinv = 1/m.
__global__ void __launch_bounds__(kBlock) l1_dinv_kernel(const int32_t* __restrict__ hdr,
                                                         const int64_t* __restrict__ ptr,
                                                         const int64_t* __restrict__ cptr,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val, int64_t n, int64_t ncols,
                                                         int lanes, const uint8_t* __restrict__ iperm,
                                                         double* __restrict__ dinv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double aii = 0.0, off = 0.0;
    bool found = false;
    if (lanes == 1) {
      const int64_t t = slot_of_row(iperm, i);
      const int64_t s = t >> 5;
      const int64_t vb = ptr[s] + (t & 31);
      const int w = (int)((ptr[s + 1] - ptr[s]) >> 5);
      for (int k = 0; k < w; ++k) {
        const int64_t c = sell_col(hdr, cptr, col, s, (int)(t & 31), i, k, ncols);
        const double v = val[vb + 32 * (int64_t)k];
        if (c == i && !found) {
          aii = v;
          found = true;
        } else {
          off += fabs(v);
        }
      }
    } else {
      for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
        const double v = val[k];
        if (col[k] == (int32_t)i && !found) {
          aii = v;
          found = true;
        } else {
          off += fabs(v);
        }
      }
    }
    dinv[i] = 1.0 / (aii + off);
  }
}

void launch_l1_dinv(psc_ctx* ctx, const Sell& A, double* dinv, cudaStream_t s) {
  if (A.n_rows == 0) return;
  l1_dinv_kernel<<<vec_grid(ctx, A.n_rows), kBlock, 0, s>>>(A.hdr, A.ptr, A.cptr, A.col, A.val, A.n_rows, A.n_cols_local,
                                                            A.lanes, A.iperm, dinv);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

__global__ void __launch_bounds__(kBlock) cg_update_kernel(int64_t n, double* __restrict__ x,
                                                           const double* __restrict__ p, double* __restrict__ r,
                                                           const double* __restrict__ q, const double* g_pq,
                                                           const double* g_num, int num_ranks, int nranks,
                                                           double* partials, unsigned int* ticket, double* out) {
  const double alpha = gsum(g_num, num_ranks) / gsum(g_pq, nranks);
  double acc[1] = {0.0};
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = tid; j < (n >> 1); j += stride) {
    double2 xv = ld2(x, j), rv = ld2(r, j);
    const double2 pv = ld2(p, j), qv = ld2(q, j);
    xv.x = xv.x + alpha * pv.x;
    xv.y = xv.y + alpha * pv.y;
    rv.x = rv.x - alpha * qv.x;
    rv.y = rv.y - alpha * qv.y;
    st2(x, j, xv);
    st2(r, j, rv);
    acc[0] += rv.x * rv.x;
    acc[0] += rv.y * rv.y;
  }
  if ((n & 1) && tid == 0) {
    const int64_t i = n - 1;
    x[i] = x[i] + alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    acc[0] += ri * ri;
  }
  grid_reduce<1>(acc, partials, ticket, out, 1);
}

void launch_cg_update(psc_ctx* ctx, int64_t n, double* x, const double* p, double* r, const double* q,
                      const double* g_pq, const double* g_num, int num_ranks, int nranks, const RedSite* red,
                      double* red_out, cudaStream_t s) {
  KtScope kts(ctx, s, "cg_update", 48.0 * n, 48.0 * n);
  PSC_REQUIRE(al16(x) && al16(p) && al16(r) && al16(q), PSC_ERR_STATE,
              "vector kernels need 16-byte aligned buffers");
  const int g = std::min(vec_grid(ctx, n), red->grid);
  launch_k(cg_update_kernel, g, kBlock, 0, s, n, x, p, r, q, g_pq, g_num, num_ranks, nranks, red->partials,
           red->ticket, red_out);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// FCG(1) (Notay; the paper's Krylov method): the new direction is
// A-orthogonalised against the previous one only, p = z - ((z, q_old) / (p_old,
// q_old)) p_old with q_old = A p_old, and alpha needs (p, r), reduced here.
__global__ void __launch_bounds__(kBlock) fcg_dir_kernel(int64_t n, const double* __restrict__ z,
                                                         double* __restrict__ p, const double* __restrict__ r,
                                                         const double* g_zq, const double* g_pq, int nranks,
                                                         double* partials, unsigned int* ticket, double* out) {
  const double beta = gsum(g_zq, nranks) / gsum(g_pq, nranks);
  double acc[1] = {0.0};
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = tid; j < (n >> 1); j += stride) {
    const double2 zv = ld2(z, j), rv = ld2(r, j);
    double2 pv = ld2(p, j);
    pv.x = zv.x - beta * pv.x;
    pv.y = zv.y - beta * pv.y;
    st2(p, j, pv);
    acc[0] += pv.x * rv.x;
    acc[0] += pv.y * rv.y;
  }
  if ((n & 1) && tid == 0) {
    const double pi = z[n - 1] - beta * p[n - 1];
    p[n - 1] = pi;
    acc[0] += pi * r[n - 1];
  }
  grid_reduce<1>(acc, partials, ticket, out, 1);
}

void launch_fcg_dir(psc_ctx* ctx, int64_t n, const double* z, double* p, const double* r, const double* g_zq,
                    const double* g_pq, int nranks, const RedSite* red, double* red_out, cudaStream_t s) {
  KtScope kts(ctx, s, "fcg_dir", 32.0 * n, 32.0 * n);
  PSC_REQUIRE(al16(z) && al16(p) && al16(r), PSC_ERR_STATE, "vector kernels need 16-byte aligned buffers");
  const int g = std::min(vec_grid(ctx, n), red->grid);
  launch_k(fcg_dir_kernel, g, kBlock, 0, s, n, z, p, r, g_zq, g_pq, nranks, red->partials, red->ticket, red_out);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// ------------------------------------------- coarsest PCG, launch-per-step form
// ("at most 40 iterations of the Preconditioned CG coupled to l1-Jacobi
// preconditioner").  The host records all maxit iterations into the iteration
// graph; `done` turns the remaining steps into no-ops once the coarse residual
// test (or a breakdown) fires.  Every CTA takes the same decision from the same
// gathered scalars, so either all CTAs enter a reduction or none does.
__device__ __forceinline__ int ld_flag(const int* f) { return *(const volatile int*)f; }

__global__ void __launch_bounds__(kBlock) cpcg_init_kernel(int64_t n, const double* __restrict__ b,
                                                           const double* __restrict__ dinv, double* __restrict__ x,
                                                           double* __restrict__ r, double* __restrict__ z,
                                                           double* __restrict__ p, int* done, double* partials,
                                                           unsigned int* ticket, double* out, int stride) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *done = 0;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = b[i];
    const double zi = dinv[i] * bi;
    x[i] = 0.0;
    r[i] = bi;
    z[i] = zi;
    p[i] = zi;
    acc[0] += bi * zi;
    acc[1] += bi * bi;
  }
  grid_reduce<2>(acc, partials, ticket, out, stride);
}

__global__ void __launch_bounds__(kBlock) cpcg_update_kernel(int64_t n, double* __restrict__ x,
                                                             const double* __restrict__ p, double* __restrict__ r,
                                                             const double* __restrict__ q, double* __restrict__ z,
                                                             const double* __restrict__ dinv, const double* g_pq,
                                                             const double* g_rz, int nr, int* done, double* partials,
                                                             unsigned int* ticket, double* out, int stride) {
  if (ld_flag(done)) return;
  const double pq = gsum(g_pq, nr);
  if (!(pq > 0.0)) {  // breakdown (or b = 0): keep x
    if (blockIdx.x == 0 && threadIdx.x == 0) *done = 1;
    return;
  }
  const double alpha = gsum(g_rz, nr) / pq;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = x[i] + alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    const double zi = dinv[i] * ri;
    r[i] = ri;
    z[i] = zi;
    acc[0] += ri * ri;
    acc[1] += ri * zi;
  }
  grid_reduce<2>(acc, partials, ticket, out, stride);
}

__global__ void __launch_bounds__(kBlock) cpcg_dir_kernel(int64_t n, const double* __restrict__ z,
                                                          double* __restrict__ p, const double* g_rr,
                                                          const double* g_bb, const double* g_rzn, const double* g_rz,
                                                          int nr, double tol, int* done) {
  if (ld_flag(done)) return;
  if (sqrt(gsum(g_rr, nr)) <= tol * sqrt(gsum(g_bb, nr))) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *done = 1;
    return;
  }
  const double beta = gsum(g_rzn, nr) / gsum(g_rz, nr);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

void launch_cpcg_init(psc_ctx* ctx, int64_t n, const double* b, const double* dinv, double* x, double* r, double* z,
                      double* p, int* done, const RedSite* red, double* out, int stride, cudaStream_t s) {
  KtScope kts(ctx, s, "cpcg_init", 40.0 * n, 40.0 * n);
  const int g = std::min(vec_grid(ctx, n), red->grid);
  launch_k(cpcg_init_kernel, g, kBlock, 0, s, n, b, dinv, x, r, z, p, done, red->partials, red->ticket, out, stride);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

void launch_cpcg_update(psc_ctx* ctx, int64_t n, double* x, const double* p, double* r, const double* q, double* z,
                        const double* dinv, const double* g_pq, const double* g_rz, int nr, int* done,
                        const RedSite* red, double* out, int stride, cudaStream_t s) {
  KtScope kts(ctx, s, "cpcg_update", 64.0 * n, 64.0 * n);
  const int g = std::min(vec_grid(ctx, n), red->grid);
  launch_k(cpcg_update_kernel, g, kBlock, 0, s, n, x, p, r, q, z, dinv, g_pq, g_rz, nr, done, red->partials,
           red->ticket, out, stride);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

void launch_cpcg_dir(psc_ctx* ctx, int64_t n, const double* z, double* p, const double* g_rr, const double* g_bb,
                     const double* g_rzn, const double* g_rz, int nr, double tol, int* done, cudaStream_t s) {
  KtScope kts(ctx, s, "cpcg_dir", 24.0 * n, 24.0 * n);
  launch_k(cpcg_dir_kernel, vec_grid(ctx, n), kBlock, 0, s, n, z, p, g_rr, g_bb, g_rzn, g_rz, nr, tol, done);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

__global__ void __launch_bounds__(kBlock) xpby_kernel(int64_t n, const double* __restrict__ z, double* __restrict__ p,
                                                      const double* g_rz, double* rz_old, int nranks,
                                                      unsigned int* ticket) {
  const double rz = gsum(g_rz, nranks);
  const double beta = rz / __ldcg(rz_old);
  // (16-byte form measured 66 vs 62 us: kept scalar; cg_update gains from it: 121 vs 164 us)
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
  KtScope kts(ctx, s, "xpby", 24.0 * n, 24.0 * n);
  PSC_REQUIRE(al16(z) && al16(p), PSC_ERR_STATE, "vector kernels need 16-byte aligned buffers");
  launch_k(xpby_kernel, vec_grid(ctx, n), kBlock, 0, s, n, z, p, g_rz, rz_old, nranks, red->ticket);
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
  KtScope kts(ctx, s, "dot", 16.0 * n, 16.0 * n);
  const int g = std::min(vec_grid(ctx, n), red->grid);
  launch_k(dot_kernel, g, kBlock, 0, s, n, a, b, red->partials, red->ticket, red_out);
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
  launch_k(pack_kernel, vec_grid(ctx, n), kBlock, 0, s, n, idx, x, sendbuf);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

__global__ void gather_kernel(int64_t n, const int64_t* __restrict__ map, const double* __restrict__ in,
                              double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[map[i]];
}

void launch_gather(psc_ctx* ctx, int64_t n, const int64_t* map, const double* in, double* out, cudaStream_t s) {
  KtScope kts(ctx, s, "gather", 24.0 * n, 24.0 * n);
  if (n == 0) return;
  launch_k(gather_kernel, vec_grid(ctx, n), kBlock, 0, s, n, map, in, out);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// ------------------------------------------------------------ coarsest solve
// One CTA runs the whole coarsest-level solver (l1-Jacobi "as coarse
// solver (30 iterations)") instead of 30 dependent launches: iterate,
// right-hand side and dinv live in shared memory and, when it fits (227 KB),
// so does A_coarse.  `gk` lanes share a row (gk = pow2floor(1024 / n), so all
// 1024 threads work on every sweep); partial sums are combined by a fixed
// shuffle tree.
constexpr int kCoarseThreads = 1024;
constexpr int kMaxSmem = 227 * 1024;
int64_t coarse_smem_rows() { return (64 * 1024) / (4 * sizeof(double)); }

struct CoarseArgs {
  const int32_t* hdr;   // sliced ELL only
  const int64_t* ptr;
  const int64_t* cptr;  // sliced ELL only
  const int32_t* col;
  const double* val;
  int64_t n, nptr, padded, col_slots;
  int gk;
  const double* dinv;
  const double* b;
  double* xout;
  int nsweeps;
  const uint8_t* iperm;  // sliced ELL: SELL-C-sigma row -> slot (nullptr: identity)
};

template <bool SELL, bool STAGE>
__global__ void __launch_bounds__(kCoarseThreads) coarse_solve(CoarseArgs a) {
  extern __shared__ double sm[];
  const int64_t n = a.n;
  double* xa = sm;
  double* xb = sm + n;
  double* bs = sm + 2 * n;
  double* ds = sm + 3 * n;
  const double* val = a.val;
  const int64_t* ptr = a.ptr;
  const int64_t* cptr = a.cptr;
  const int32_t* col = a.col;
  if constexpr (STAGE) {
    double* v_s = sm + 4 * n;
    int64_t* p_s = reinterpret_cast<int64_t*>(v_s + a.padded);
    int64_t* cp_s = p_s + a.nptr;
    int32_t* c_s = reinterpret_cast<int32_t*>(cp_s + (SELL ? a.nptr : 0));
    for (int64_t k = threadIdx.x; k < a.padded; k += blockDim.x) v_s[k] = a.val[k];
    for (int64_t k = threadIdx.x; k < a.col_slots; k += blockDim.x) c_s[k] = a.col[k];
    for (int64_t k = threadIdx.x; k < a.nptr; k += blockDim.x) {
      p_s[k] = a.ptr[k];
      if constexpr (SELL) cp_s[k] = a.cptr[k];
    }
    val = v_s;
    ptr = p_s;
    cptr = cp_s;
    col = c_s;
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    bs[i] = a.b[i];
    ds[i] = a.dinv[i];
    xa[i] = (a.nsweeps > 0) ? ds[i] * bs[i] : 0.0;  // first sweep from x = 0
  }
  __syncthreads();
  const int gk = a.gk;
  const int sub = threadIdx.x & (gk - 1);
  const int rows_per_pass = kCoarseThreads / gk;
  for (int sw = 1; sw < a.nsweeps; ++sw) {
    for (int64_t r0 = 0; r0 < n; r0 += rows_per_pass) {
      const int64_t i = r0 + threadIdx.x / gk;
      double sum = 0.0;
      if (i < n) {
        if constexpr (SELL) {
          const int64_t t = slot_of_row(a.iperm, i);
          const int64_t s = t >> 5;
          const int64_t base = ptr[s] + (t & 31);
          const int w = (int)((ptr[s + 1] - ptr[s]) >> 5);
          for (int k = sub; k < w; k += gk) {
            const int64_t c = sell_col(a.hdr, cptr, col, s, (int)(t & 31), i, k, n);
            if (c >= 0) sum = fma(val[base + 32 * k], xa[c], sum);
          }
        } else {
          const int64_t base = ptr[i];
          const int w = (int)(ptr[i + 1] - base);
          for (int k = sub; k < w; k += gk) sum = fma(val[base + k], xa[col[base + k]], sum);
        }
      }
      for (int o = gk / 2; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o, gk);
      if (sub == 0 && i < n) xb[i] = xa[i] + ds[i] * (bs[i] - sum);
    }
    __syncthreads();
    double* t = xa;
    xa = xb;
    xb = t;
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a.xout[i] = xa[i];
}

template <bool SELL, bool STAGE>
static void coarse_launch(const CoarseArgs& a, size_t smem, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    PSC_CUDA(cudaFuncSetAttribute(coarse_solve<SELL, STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    attr = true;
  }
  launch_k(coarse_solve<SELL, STAGE>, 1, kCoarseThreads, smem, s, a);
}

// The one-CTA solver pays off only when A_coarse is staged in shared memory; a
// larger coarsest level (e.g. 602 rows x ~600 nnz on the 1e4-jump problem:
// 11 ms per call from L2 in one CTA) runs as full-grid sweep launches instead.
bool coarse_one_cta_fits(const Sell& A) {
  const int64_t n = A.n_rows;
  const int64_t nptr = A.lanes == 1 ? A.n_units + 1 : n + 1;
  const size_t vec = (size_t)std::max<int64_t>(n, 1) * 4 * sizeof(double);
  const size_t mat = (size_t)A.padded * sizeof(double) + (size_t)A.col_slots * sizeof(int32_t) +
                     (size_t)nptr * sizeof(int64_t) * (A.lanes == 1 ? 2 : 1);
  return n <= coarse_smem_rows() && vec + mat <= (size_t)kMaxSmem;
}

void launch_coarse_solve(psc_ctx* ctx, const Sell& A, const double* dinv, const double* b, double* x, int nsweeps,
                         cudaStream_t s) {
  KtScope kts(ctx, s, "coarse_solve", 12.0 * (double)A.nnz + 24.0 * (double)A.n_rows,
               8.0 * (double)A.padded + 4.0 * (double)A.col_slots + 24.0 * (double)A.n_rows);
  const int64_t n = A.n_rows;
  PSC_REQUIRE(n <= coarse_smem_rows(), PSC_ERR_STATE, "coarsest level too large for the one-CTA solver");
  PSC_REQUIRE(A.n_cols_local == n, PSC_ERR_STATE, "coarsest matrix must have no halo");
  const bool sell = (A.lanes == 1);
  const int64_t nptr = sell ? A.n_units + 1 : n + 1;
  int gk = 1;
  while (gk < 32 && (int64_t)(gk * 2) * std::max<int64_t>(n, 1) <= kCoarseThreads) gk *= 2;
  CoarseArgs a{A.hdr, A.ptr, A.cptr, A.col, A.val, n, nptr, A.padded, A.col_slots, gk, dinv, b, x, nsweeps, A.iperm};
  const size_t vec = (size_t)std::max<int64_t>(n, 1) * 4 * sizeof(double);
  const size_t mat = (size_t)A.padded * sizeof(double) + (size_t)A.col_slots * sizeof(int32_t) +
                     (size_t)nptr * sizeof(int64_t) * (sell ? 2 : 1);
  const bool stage = vec + mat <= (size_t)kMaxSmem;
  const size_t smem = stage ? vec + mat : vec;
  if (sell) stage ? coarse_launch<true, true>(a, smem, s) : coarse_launch<true, false>(a, smem, s);
  else stage ? coarse_launch<false, true>(a, smem, s) : coarse_launch<false, false>(a, smem, s);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// Dense coarsest solver: the coarsest A (nearly dense after Galerkin
// coarsening: ~115 of 141 entries per row on 256^3) is expanded once into a
// row-major n x n array; each sweep is then a shared-memory dense matvec by
// all 1024 threads (gk lanes per row, fixed shuffle tree).
int64_t coarse_dense_max_rows() { return 144; }

__global__ void dense_from_sell_kernel(const int32_t* __restrict__ hdr, const int64_t* __restrict__ ptr,
                                       const int64_t* __restrict__ cptr,
                                       const int32_t* __restrict__ col, const double* __restrict__ val, int64_t n,
                                       int lanes, const uint8_t* __restrict__ iperm, double* __restrict__ dense) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* row = dense + i * n;
  if (lanes == 1) {
    const int64_t t = slot_of_row(iperm, i);
    const int64_t s = t >> 5;
    const int64_t vb = ptr[s] + (t & 31);
    const int w = (int)((ptr[s + 1] - ptr[s]) >> 5);
    for (int k = 0; k < w; ++k) {
      const int64_t c = sell_col(hdr, cptr, col, s, (int)(t & 31), i, k, n);
      if (c >= 0) row[c] += val[vb + 32 * (int64_t)k];  // padding adds 0.0
    }
  } else {
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) row[col[k]] += val[k];
  }
}

void dense_from_sell(psc_ctx* ctx, const Sell& A, double* dense, cudaStream_t s) {
  const int64_t n = A.n_rows;
  PSC_CUDA(cudaMemsetAsync(dense, 0, sizeof(double) * n * n, s));
  if (n == 0) return;
  dense_from_sell_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(A.hdr, A.ptr, A.cptr, A.col, A.val, n, A.lanes,
                                                                      A.iperm, dense);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// Register-blocked: warp w owns rows w + 24 m (m < 6), lane owns columns
// lane + 32 c (c < 5), so n <= 144: A_coarse lives in registers (30 doubles per thread)
// for all sweeps; each sweep reads x from shared memory, does 25 FMAs per
// thread and one xor-butterfly per row (fixed order, every lane gets the sum).
constexpr int kCR = 6, kCC = 5, kDenseWarps = 24;  // 24 warps x 6 rows = 144 rows, 32 lanes x 5 cols = 160
__global__ void __launch_bounds__(kDenseWarps * 32, 1) coarse_dense(const double* __restrict__ Ad, int n,
                                                                  const double* __restrict__ dinv,
                                                                  const double* __restrict__ b,
                                                                  double* __restrict__ xout, int nsweeps, int gk_unused) {
  __shared__ double xs[2][32 * kCC];
  __shared__ double bs[32 * kCC], ds[32 * kCC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double a[kCR][kCC];
#pragma unroll
  for (int m = 0; m < kCR; ++m) {
    const int i = w + kDenseWarps * m;
#pragma unroll
    for (int c = 0; c < kCC; ++c) {
      const int j = lane + 32 * c;
      a[m][c] = (i < n && j < n) ? __ldg(Ad + (size_t)i * n + j) : 0.0;
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    bs[i] = b[i];
    ds[i] = dinv[i];
    xs[0][i] = (nsweeps > 0) ? ds[i] * bs[i] : 0.0;  // first sweep from x = 0
  }
  __syncthreads();
  int cur = 0;
  for (int sw = 1; sw < nsweeps; ++sw) {
    double xj[kCC];
#pragma unroll
    for (int c = 0; c < kCC; ++c) {
      const int j = lane + 32 * c;
      xj[c] = j < n ? xs[cur][j] : 0.0;
    }
#pragma unroll
    for (int m = 0; m < kCR; ++m) {
      double sum = 0.0;
#pragma unroll
      for (int c = 0; c < kCC; ++c) sum = fma(a[m][c], xj[c], sum);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const int i = w + kDenseWarps * m;
      if (lane == m && i < n) xs[cur ^ 1][i] = xs[cur][i] + ds[i] * (bs[i] - sum);
    }
    __syncthreads();
    cur ^= 1;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) xout[i] = xs[cur][i];
}

void launch_coarse_dense(psc_ctx* ctx, const double* Ad, int64_t n, const double* dinv, const double* b, double* x,
                         int nsweeps, cudaStream_t s) {
  KtScope kts(ctx, s, "coarse_dense", 8.0 * n * n + 24.0 * n, 8.0 * n * n + 24.0 * n);
  PSC_REQUIRE(n <= coarse_dense_max_rows(), PSC_ERR_STATE, "coarsest level too large for the dense solver");
  launch_k(coarse_dense, 1, kDenseWarps * 32, 0, s, Ad, (int)n, dinv, b, x, nsweeps, 0);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// Dense one-CTA coarsest PCG with the l1-Jacobi preconditioner, same
// register blocking of A as coarse_dense for q = A p (all 24 warps, p from
// shared memory); the vector recurrences and the fixed-order reductions
// (per-lane partials over c = 0..4, then an xor butterfly) run in warp 0 with
// x, r, p, dinv in shared memory; two CTA barriers per iteration.  The stop
// decision (||r|| <= tol ||b||, or p^T A p <= 0) is taken by warp 0 and read by
// all warps after a barrier.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kDenseWarps * 32, 1) coarse_dense_pcg(const double* __restrict__ Ad, int n,
                                                                      const double* __restrict__ dinv,
                                                                      const double* __restrict__ b,
                                                                      double* __restrict__ xout, int maxit,
                                                                      double tol) {
  constexpr int V = 32 * kCC;
  __shared__ double ps[V], qs[V], xs[V], rs[V], ds[V];
  __shared__ int stop_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double a[kCR][kCC];
#pragma unroll
  for (int m = 0; m < kCR; ++m) {
    const int i = w + kDenseWarps * m;
#pragma unroll
    for (int c = 0; c < kCC; ++c) {
      const int j = lane + 32 * c;
      a[m][c] = (i < n && j < n) ? __ldg(Ad + (size_t)i * n + j) : 0.0;
    }
  }
  double rz = 0.0, nb = 0.0;  // warp 0
  if (w == 0) {
    double rz_l = 0.0, bb_l = 0.0;
#pragma unroll
    for (int c = 0; c < kCC; ++c) {
      const int j = lane + 32 * c;
      const double bj = j < n ? b[j] : 0.0;
      const double dj = j < n ? dinv[j] : 0.0;
      const double zj = dj * bj;
      xs[j] = 0.0;
      rs[j] = bj;
      ds[j] = dj;
      ps[j] = zj;
      qs[j] = 0.0;
      rz_l += bj * zj;
      bb_l += bj * bj;
    }
    rz = warp_sum(rz_l);
    nb = sqrt(warp_sum(bb_l));
    if (lane == 0) stop_s = !(nb > 0.0);
  }
  __syncthreads();
  for (int k = 1; k <= maxit; ++k) {
    if (stop_s) break;
    // q = A p
    double pj[kCC];
#pragma unroll
    for (int c = 0; c < kCC; ++c) pj[c] = ps[lane + 32 * c];
#pragma unroll
    for (int m = 0; m < kCR; ++m) {
      double sum = 0.0;
#pragma unroll
      for (int c = 0; c < kCC; ++c) sum = fma(a[m][c], pj[c], sum);
      sum = warp_sum(sum);
      const int i = w + kDenseWarps * m;
      if (lane == m && i < n) qs[i] = sum;
    }
    __syncthreads();
    if (w == 0) {
      double pq_l = 0.0;
#pragma unroll
      for (int c = 0; c < kCC; ++c) pq_l += ps[lane + 32 * c] * qs[lane + 32 * c];
      const double pq = warp_sum(pq_l);
      int stop = 0;
      if (!(pq > 0.0)) {
        stop = 1;  // breakdown: keep x
      } else {
        const double alpha = rz / pq;
        double rr_l = 0.0;
#pragma unroll
        for (int c = 0; c < kCC; ++c) {
          const int j = lane + 32 * c;
          xs[j] = xs[j] + alpha * ps[j];
          const double rj = rs[j] - alpha * qs[j];
          rs[j] = rj;
          rr_l += rj * rj;
        }
        if (sqrt(warp_sum(rr_l)) <= tol * nb) {
          stop = 1;
        } else {
          double rz_l = 0.0;
#pragma unroll
          for (int c = 0; c < kCC; ++c) {
            const int j = lane + 32 * c;
            rz_l += rs[j] * (ds[j] * rs[j]);
          }
          const double rzn = warp_sum(rz_l);
          const double beta = rzn / rz;
          rz = rzn;
#pragma unroll
          for (int c = 0; c < kCC; ++c) {
            const int j = lane + 32 * c;
            ps[j] = ds[j] * rs[j] + beta * ps[j];
          }
        }
      }
      if (lane == 0) stop_s = stop;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) xout[i] = xs[i];
}

void launch_coarse_dense_pcg(psc_ctx* ctx, const double* Ad, int64_t n, const double* dinv, const double* b,
                             double* x, int maxit, double tol, cudaStream_t s) {
  KtScope kts(ctx, s, "coarse_dense_pcg", 8.0 * n * n + 24.0 * n, 8.0 * n * n + 24.0 * n);
  PSC_REQUIRE(n <= coarse_dense_max_rows(), PSC_ERR_STATE, "coarsest level too large for the dense solver");
  launch_k(coarse_dense_pcg, 1, kDenseWarps * 32, 0, s, Ad, (int)n, dinv, b, x, maxit, tol);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

// Row bandwidth of a square matrix in the sliced-ELL layout: max |j - i| over
// the stored entries (DIA slices: their offsets; ELL padding repeats a real
// column of the row, an empty row pads with column 0 — conservative).
// -------------------------------------------------- dense suffix operator
// y = D b for a dense row-major n x n operator (the V-cycle of the deepest
// levels precomputed as a matrix, hier.cu): one warp per row, b staged in
// shared memory, four accumulators over column blocks (fixed order), xor tree.
__global__ void __launch_bounds__(256) dense_gemv_kernel(const double* __restrict__ D, int64_t n,
                                                         const double* __restrict__ b, double* __restrict__ y) {
  extern __shared__ double bs[];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) bs[i] = b[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (row < n) {
    const double* Dr = D + row * n;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t j = lane;
    for (; j + 96 < n; j += 128) {
      s0 = fma(__ldg(Dr + j), bs[j], s0);
      s1 = fma(__ldg(Dr + j + 32), bs[j + 32], s1);
      s2 = fma(__ldg(Dr + j + 64), bs[j + 64], s2);
      s3 = fma(__ldg(Dr + j + 96), bs[j + 96], s3);
    }
    for (; j < n; j += 32) s0 = fma(__ldg(Dr + j), bs[j], s0);
    double sum = (s0 + s1) + (s2 + s3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) y[row] = sum;
  }
}

int64_t dense_gemv_max_rows() { return 6144; }  // b in 48 KB of shared memory

void launch_dense_gemv(psc_ctx* ctx, const double* D, int64_t n, const double* b, double* y, cudaStream_t s) {
  KtScope kts(ctx, s, "dense_gemv", 8.0 * n * n + 16.0 * n, 8.0 * n * n + 16.0 * n);
  PSC_REQUIRE(n >= 1 && n <= dense_gemv_max_rows(), PSC_ERR_STATE, "dense operator too large");
  launch_k(dense_gemv_kernel, (unsigned)((n + 7) / 8), 256, (size_t)n * sizeof(double), s, D, n, b, y);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}

__global__ void transpose_kernel(const double* __restrict__ in, int64_t n, double* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n * n) return;
  const int64_t i = k / n, j = k - i * n;
  out[i * n + j] = in[j * n + i];
}

void launch_transpose(psc_ctx* ctx, const double* in, int64_t n, double* out, cudaStream_t s) {
  transpose_kernel<<<(unsigned)((n * n + 255) / 256), 256, 0, s>>>(in, n, out);
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


// One warp per slice: width (max row length), off-rank flag, nnz, and — when
// allowed and every column is owned — the sorted distinct diagonal offsets
// (local col - local row) of the slice, found by repeated warp-min over the
// rows' sorted column lists.  The slice is stored DIA when d <= 1.5 w
// (8 B x 32 d value slots beat 12 B x 32 w value+column slots).
__global__ void sell_width_kernel(int64_t n_rows, int64_t n_slices, const int64_t* __restrict__ rowptr,
                                  const int64_t* __restrict__ colg, int64_t own_begin, int64_t n_own, int allow_dia,
                                  int max_dia, int allow16, const uint8_t* __restrict__ perm,
                                  int64_t* __restrict__ vslots, int64_t* __restrict__ cslots,
                                  int64_t* __restrict__ snnz, int32_t* __restrict__ bflag, int32_t* __restrict__ dia_d,
                                  int32_t* __restrict__ dia_off, int32_t* __restrict__ e16) {
  const int lane = threadIdx.x & 31;
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_slices) return;
  const int64_t i = row_of_slot(perm, s * 32 + lane);  // (allow_dia == 0 when perm is set)
  int len = 0, off = 0;
  int64_t b = 0;
  if (i < n_rows) {
    b = rowptr[i];
    const int64_t e = rowptr[i + 1];
    len = (int)(e - b);
    for (int64_t k = b; k < e; ++k) {
      const int64_t g = colg[k];
      off |= (g < own_begin || g >= own_begin + n_own);
    }
  }
  int w = len, tot = len;
  for (int o = 16; o > 0; o >>= 1) {
    w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
    tot += __shfl_xor_sync(0xffffffffu, tot, o);
  }
  off = __any_sync(0xffffffffu, off);
  int d = 0;
  if (allow_dia && !off && w > 0 && w <= max_dia) {
    int q = 0;
    bool ok = true;
    for (;;) {
      const long long my = (q < len) ? (long long)(colg[b + q] - own_begin - i) : LLONG_MAX;
      long long mn = my;
      for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      if (mn == LLONG_MAX) break;
      if (d == max_dia) {
        ok = false;
        break;
      }
      if (lane == 0) dia_off[s * kMaxDia + d] = (int32_t)mn;
      ++d;
      if (my == mn) ++q;
    }
    if (!ok || 2 * d > 3 * w) d = 0;
  }
  // ELL slice of at most kTmaMaxW columns, all owned, spanning < 2^16: uint16 offsets
  // from the smallest.  (Wider slices keep int32 columns: on the level-1 operator of
  // 256^3, ~31 per row, 16-bit offsets made the thread-per-row sweep slower, 166 vs
  // 161 us, while P_0 in the TMA kernel gained 204 vs 215 us.)
  int base = -1;
  if (allow16 && d == 0 && !off && w > 0 && w <= kTmaMaxW) {
    long long mn = LLONG_MAX, mx = LLONG_MIN;
    for (int q = 0; q < len; ++q) {
      const long long c = (long long)(colg[b + q] - own_begin);
      mn = min(mn, c);
      mx = max(mx, c);
    }
    for (int o = 16; o > 0; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (mx - mn < 65536) base = (int)mn;
  }
  if (lane == 0) {
    vslots[s] = 32 * (int64_t)(d ? d : w);
    // DIA: offsets, padded to 16 B; ELL: int32 columns; ELL16: uint16 columns
    cslots[s] = d ? (int64_t)((d + 3) & ~3) : (base >= 0 ? 16 * (int64_t)w : 32 * (int64_t)w);
    e16[s] = base;
    snnz[s] = tot;
    bflag[s] = off;
    dia_d[s] = d;
  }
}

// thread per row: scatter the row into its slice column-major, renumbering
// columns (ELL slice) or aligning it with the slice's diagonals (DIA slice)
__global__ void sell_fill_kernel(int64_t n_rows, int64_t n_slices, const int64_t* __restrict__ rowptr,
                                 const int64_t* __restrict__ colg, const double* __restrict__ valcsr,
                                 const int64_t* __restrict__ ptr, const int64_t* __restrict__ cptr,
                                 const int32_t* __restrict__ dia_d, const int32_t* __restrict__ dia_off,
                                 const int32_t* __restrict__ e16, int64_t own_begin, int64_t n_own,
                                 const int64_t* __restrict__ halo, int64_t nh, const uint8_t* __restrict__ perm,
                                 int32_t* __restrict__ col, double* __restrict__ val, int64_t* __restrict__ slot,
                                 int* err) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // slot
  if (t >= n_slices * 32) return;
  const int64_t s = t >> 5;
  const int lane = (int)(t & 31);
  const int64_t i = row_of_slot(perm, t);  // row held by the slot
  const int64_t vb = ptr[s], cb = cptr[s];
  const int w = (int)((ptr[s + 1] - vb) >> 5);
  int64_t b = 0, e = 0;
  if (i < n_rows) {
    b = rowptr[i];
    e = rowptr[i + 1];
  }
  const int d = dia_d[s];
  if (d > 0) {
    int64_t q = b;
    for (int j = 0; j < d; ++j) {
      const int32_t o = dia_off[s * kMaxDia + j];
      double v = 0.0;
      if (q < e && colg[q] - own_begin == i + o) {
        v = valcsr[q];
        if (slot) slot[q] = vb + 32 * (int64_t)j + lane;
        ++q;
      }
      val[vb + 32 * (int64_t)j + lane] = v;
      if (lane == 0) col[cb + j] = o;
    }
    if (lane == 0)
      for (int j = d; j < ((d + 3) & ~3); ++j) col[cb + j] = 0;
    if (q != e) *err = 2;
    return;
  }
  const int32_t base = e16[s];
  if (base >= 0) {  // kEll16 (every column owned: col - own_begin - base in [0, 2^16))
    uint16_t* c16 = reinterpret_cast<uint16_t*>(col + cb);
    uint16_t last = 0;
    for (int k = 0; k < w; ++k) {
      const int64_t o = 32 * (int64_t)k + lane;
      if (b + k < e) {
        const int64_t c = colg[b + k] - own_begin - base;
        if (c < 0 || c > 65535) *err = 1;
        last = (uint16_t)c;
        val[vb + o] = valcsr[b + k];
        if (slot) slot[b + k] = vb + o;
      } else {
        val[vb + o] = 0.0;
      }
      c16[o] = last;
    }
    return;
  }
  int32_t last = 0;
  for (int k = 0; k < w; ++k) {
    const int64_t o = 32 * (int64_t)k + lane;
    if (b + k < e) {
      last = map_col(colg[b + k], own_begin, n_own, halo, nh, err);
      col[cb + o] = last;
      val[vb + o] = valcsr[b + k];
      if (slot) slot[b + k] = vb + o;
    } else {
      col[cb + o] = last;
      val[vb + o] = 0.0;
    }
  }
}

// SELL-C-sigma order of one 256-row window (one CTA of kSortWin threads): rows by
// decreasing length, ties by increasing row index (a stable order, so the layout
// is deterministic).  perm[slot] = row offset, iperm[row] = slot offset.
__global__ void __launch_bounds__(kSortWin) sell_sort_kernel(int64_t n_rows, const int64_t* __restrict__ rowptr,
                                                             uint8_t* __restrict__ perm, uint8_t* __restrict__ iperm) {
  __shared__ int len[kSortWin];
  const int64_t w0 = (int64_t)blockIdx.x * kSortWin;
  const int me = threadIdx.x;
  const int64_t i = w0 + me;
  const int mine = i < n_rows ? (int)(rowptr[i + 1] - rowptr[i]) : -1;  // absent rows last
  len[me] = mine;
  __syncthreads();
  int rank = 0;
  for (int j = 0; j < kSortWin; ++j) {
    const int lj = len[j];
    rank += (lj > mine) || (lj == mine && j < me);
  }
  perm[w0 + rank] = (uint8_t)me;
  iperm[w0 + me] = (uint8_t)rank;
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
                               double* __restrict__ val, int64_t* __restrict__ slot, int* err) {
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
      if (slot) slot[b + k] = o0 + k;
    } else {
      col[o0 + k] = last;
      val[o0 + k] = 0.0;
    }
  }
}

// Layout choice: rows shorter than PSC_RG_MIN = 100 on average ->
// sliced ELL, thread per row (measured faster than row groups on the 31-nnz/row
// level-1 operator of 256^3: 150 vs 179 us per sweep); long rows -> G lanes per
// row, G = pow2floor(mean / PSC_RG_DIV) clamped to [4, 32].  PSC_LANES forces a
// layout (1, 4, 8, 16, 32).
int choose_lanes(int64_t n_rows, int64_t nnz) {
  const int forced = env_int("PSC_LANES", 0);
  if (forced == 1 || forced == 4 || forced == 8 || forced == 16 || forced == 32) return forced;
  const double mu = n_rows ? (double)nnz / (double)n_rows : 0.0;
  // small (L2-resident) matrices with longer rows: thread-per-row slices leave too few
  // warps per SM to cover the gather latency (level 2 of 256^3: 65,000 rows, 2,031
  // warps for 148 SMs); row groups of G = mu / PSC_RG_SMALL_DIV lanes spread a row over
  // a group (experiment: PSC_RG_SMALL_MB = size limit in MB, 0 = off)
  const int small_mb = env_int("PSC_RG_SMALL_MB", 0);
  if (small_mb > 0 && mu >= 16 && 12.0 * (double)nnz <= (double)small_mb * 1048576.0) {
    const double t = mu / std::max(1, env_int("PSC_RG_SMALL_DIV", 8));
    int G = 4;
    while (G * 2 <= t && G < 32) G *= 2;
    return G;
  }
  if (mu < env_int("PSC_RG_MIN", 100)) return 1;
  const double t = mu / std::max(1, env_int("PSC_RG_DIV", 1));
  int G = 4;
  while (G * 2 <= t && G < 32) G *= 2;
  return G;
}

__global__ void sell_hdr_kernel(int64_t n_slices, const int64_t* __restrict__ ptr, const int64_t* __restrict__ cptr,
                                const int32_t* __restrict__ dia_d, const int32_t* __restrict__ dia_off,
                                const int32_t* __restrict__ e16, int32_t* __restrict__ hdr) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_slices) return;
  int32_t* h = hdr + s * kHdr;
  const int64_t vb = ptr[s], cb = cptr[s];
  h[0] = (int32_t)(uint32_t)(vb & 0xffffffffu);
  h[1] = (int32_t)(uint32_t)((uint64_t)vb >> 32);
  h[2] = (int32_t)(uint32_t)(cb & 0xffffffffu);
  h[3] = (int32_t)(uint32_t)((uint64_t)cb >> 32);
  h[4] = (int32_t)((ptr[s + 1] - vb) >> 5);
  const int d = dia_d[s];
  h[5] = d > 0 ? kDia : kEll;
  int j0 = -1;
  for (int j = 0; j < kMaxDiaHdr; ++j) h[6 + j] = j < d ? dia_off[s * kMaxDia + j] : 0;
  for (int j = 0; j < d; ++j)
    if (dia_off[s * kMaxDia + j] == 0) j0 = j;
  h[14] = j0;  // DIA: slot of the diagonal (offset 0), -1 if none
  h[15] = 0;
  if (d == 0 && e16[s] >= 0) {
    h[5] = kEll16;
    h[6] = e16[s];  // base column
  }
}

void sell_from_csr(psc_ctx* ctx, int64_t n_rows, const int64_t* d_rowptr, const int64_t* d_colg, const double* d_val,
                   int64_t nnz, int64_t own_begin, int64_t n_own, const int64_t* d_halo, int64_t n_halo, Sell& S,
                   cudaStream_t s, int lanes, bool allow_dia) {
  S.n_rows = n_rows;
  S.n_cols_local = n_own + n_halo;
  S.nnz = nnz;
  // value slot of every CSR entry (psc_mat_update_values: same structure, new values)
  S.slot = dalloc<int64_t>(nnz);
  S.lanes = lanes > 0 ? lanes : choose_lanes(n_rows, nnz);
  if (env_int("PSC_NO_DIA", 0)) allow_dia = false;
  const int RU = S.rows_per_unit();
  S.n_units = (n_rows + RU - 1) / RU;
  const bool sell = (S.lanes == 1);
  const int64_t nu = S.n_units;
  const int64_t nptr = sell ? nu + 1 : n_rows + 1;
  int* d_err = dalloc<int>(1);
  PSC_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  std::vector<int32_t> flag;      // per unit (sell) or per row (row groups)
  std::vector<int64_t> hp;        // ptr on the host
  std::vector<int32_t> hdia;      // DIA widths per slice
  std::vector<int64_t> hsnnz;     // nnz per slice
  size_t tmp_bytes = 0;
  if (sell) {
    int64_t* d_vs = dalloc<int64_t>(nu + 1);
    int64_t* d_cs = dalloc<int64_t>(nu + 1);
    int64_t* d_snnz = dalloc<int64_t>(nu);
    int32_t* d_flag = dalloc<int32_t>(nu);
    int32_t* d_diad = dalloc<int32_t>(nu);
    int32_t* d_diaoff = dalloc<int32_t>((size_t)nu * kMaxDia);
    int32_t* d_e16 = dalloc<int32_t>(nu);
    // ELL slices with 16-bit column offsets (PSC_COL16=0: 32-bit columns everywhere)
    int allow16 = env_int("PSC_COL16", 1) ? 1 : 0;
    // DIA slices with up to 8 diagonals (offsets in the slice header; A_0).  Wider DIA
    // slices (up to kMaxDia, offsets in the column region) are opt-in, PSC_DIA_MAX=64:
    // on the level-1 Galerkin operator of 256^3 they measured slower (175 vs 154 us per
    // sweep: more gathers per row for the zeros of the diagonals than ELL's padding)
    const int max_dia = std::max(1, std::min(kMaxDia, env_int("PSC_DIA_MAX", kMaxDiaHdr)));
    auto widths = [&](bool dia, const uint8_t* perm) {
      PSC_CUDA(cudaMemsetAsync(d_vs, 0, sizeof(int64_t) * (nu + 1), s));
      PSC_CUDA(cudaMemsetAsync(d_cs, 0, sizeof(int64_t) * (nu + 1), s));
      if (nu > 0) {
        sell_width_kernel<<<(unsigned)((nu * 32 + 255) / 256), 256, 0, s>>>(
            n_rows, nu, d_rowptr, d_colg, own_begin, n_own, dia ? 1 : 0, max_dia, allow16, perm, d_vs, d_cs, d_snnz,
            d_flag, d_diad, d_diaoff, d_e16);
        PSC_CUDA(cudaGetLastError());
      }
      if (!S.ptr) S.ptr = dalloc<int64_t>(nu + 1);
      if (!S.cptr) S.cptr = dalloc<int64_t>(nu + 1);
      size_t tb = 0;
      PSC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, d_vs, S.ptr, nu + 1, s));
      void* d_tmp = dalloc<char>(tb);
      PSC_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tb, d_vs, S.ptr, nu + 1, s));
      PSC_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tb, d_cs, S.cptr, nu + 1, s));
      PSC_CUDA(cudaMemcpyAsync(&S.padded, S.ptr + nu, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      PSC_CUDA(cudaMemcpyAsync(&S.col_slots, S.cptr + nu, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      hdia.resize(nu);
      if (nu) PSC_CUDA(cudaMemcpyAsync(hdia.data(), d_diad, sizeof(int32_t) * nu, cudaMemcpyDeviceToHost, s));
      PSC_CUDA(cudaStreamSynchronize(s));
      dfree(d_tmp);
    };
    widths(allow_dia, nullptr);
    // 16-bit column slices only in matrices the TMA kernel takes whole (every slice at most
    // kTmaMaxW wide): elsewhere they would send the thread-per-row kernels to their wider
    // 16-bit instantiation (P_1 of 256^3: 68 vs 64 us)
    if (allow16 && nu > 0) {
      std::vector<int64_t> hv(nu + 1);
      PSC_CUDA(cudaMemcpy(hv.data(), S.ptr, sizeof(int64_t) * (nu + 1), cudaMemcpyDeviceToHost));
      int64_t wmax = 0;
      for (int64_t u = 0; u < nu; ++u) wmax = std::max<int64_t>(wmax, (hv[u + 1] - hv[u]) / 32);
      if (wmax > kTmaMaxW) {
        allow16 = 0;
        widths(allow_dia, nullptr);
      }
    }
    // SELL-C-sigma, opt-in PSC_SORT=1: a matrix with no DIA slice whose
    // slices pad more than 2% is re-laid out with its rows sorted by length inside
    // 256-row windows (P_0 of 256^3: 1.36 -> 1.09 padded slots per stored value).
    // Measured slower on B200 (P_0 210 vs 203 us, level-1 sweep 159 vs 150 us): the
    // sorted lanes no longer touch consecutive rows, so the x gathers and the row
    // vectors lose their coalescing, which costs more than the padding saved.
    const bool any_dia = std::any_of(hdia.begin(), hdia.end(), [](int32_t d) { return d > 0; });
    if (!any_dia && env_int("PSC_SORT", 0) && (double)S.padded > 1.02 * (double)nnz && nu > 0) {
      const int64_t nwin = (nu * 32 + kSortWin - 1) / kSortWin;
      S.perm = dalloc<uint8_t>(nwin * kSortWin);
      S.iperm = dalloc<uint8_t>(nwin * kSortWin);
      sell_sort_kernel<<<(unsigned)nwin, kSortWin, 0, s>>>(n_rows, d_rowptr, S.perm, S.iperm);
      PSC_CUDA(cudaGetLastError());
      widths(false, S.perm);
    }
    S.col = dalloc<int32_t>(S.col_slots);
    S.val = dalloc<double>(S.padded);
    S.hdr = dalloc<int32_t>((size_t)nu * kHdr);
    if (nu > 0) {
      sell_fill_kernel<<<(unsigned)((nu * 32 + 255) / 256), 256, 0, s>>>(
          n_rows, nu, d_rowptr, d_colg, d_val, S.ptr, S.cptr, d_diad, d_diaoff, d_e16, own_begin, n_own, d_halo,
          n_halo, S.perm, S.col, S.val, S.slot, d_err);
      PSC_CUDA(cudaGetLastError());
      sell_hdr_kernel<<<(unsigned)((nu + 255) / 256), 256, 0, s>>>(nu, S.ptr, S.cptr, d_diad, d_diaoff, d_e16,
                                                                     S.hdr);
      PSC_CUDA(cudaGetLastError());
    }
    flag.resize(nu);
    hp.resize(nu + 1);
    hsnnz.resize(nu);
    std::vector<int32_t> he16(nu);
    if (nu) {
      PSC_CUDA(cudaMemcpyAsync(he16.data(), d_e16, sizeof(int32_t) * nu, cudaMemcpyDeviceToHost, s));
      PSC_CUDA(cudaMemcpyAsync(flag.data(), d_flag, sizeof(int32_t) * nu, cudaMemcpyDeviceToHost, s));
      PSC_CUDA(cudaMemcpyAsync(hsnnz.data(), d_snnz, sizeof(int64_t) * nu, cudaMemcpyDeviceToHost, s));
    }
    PSC_CUDA(cudaMemcpyAsync(hp.data(), S.ptr, sizeof(int64_t) * (nu + 1), cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    S.n_e16 = std::count_if(he16.begin(), he16.end(), [&](int32_t b) { return b >= 0; });
    dfree(d_snnz);
    dfree(d_flag);
    dfree(d_diad);
    dfree(d_diaoff);
    dfree(d_e16);
  } else {
    int64_t* d_len = dalloc<int64_t>(nptr);
    int32_t* d_flag = dalloc<int32_t>(n_rows);
    PSC_CUDA(cudaMemsetAsync(d_len, 0, sizeof(int64_t) * nptr, s));
    if (n_rows > 0) {
      rg_len_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, s>>>(n_rows, S.lanes, d_rowptr, d_colg, own_begin,
                                                                      n_own, d_len, d_flag);
      PSC_CUDA(cudaGetLastError());
    }
    S.ptr = dalloc<int64_t>(nptr + 2);  // +2: TMA copies of the last chunk's row pointers round up to 16 B
    PSC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_len, S.ptr, nptr, s));
    void* d_tmp = dalloc<char>(tmp_bytes);
    PSC_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_len, S.ptr, nptr, s));
    PSC_CUDA(cudaMemcpyAsync(&S.padded, S.ptr + nptr - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    dfree(d_tmp);
    dfree(d_len);
    S.col_slots = S.padded;
    S.col = dalloc<int32_t>(S.col_slots);
    S.val = dalloc<double>(S.padded);
    if (n_rows > 0) {
      rg_fill_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, s>>>(n_rows, d_rowptr, d_colg, d_val, S.ptr,
                                                                       own_begin, n_own, d_halo, n_halo, S.col,
                                                                       S.val, S.slot, d_err);
      PSC_CUDA(cudaGetLastError());
    }
    flag.resize(n_rows);
    hp.resize(nptr);
    if (n_rows) PSC_CUDA(cudaMemcpyAsync(flag.data(), d_flag, sizeof(int32_t) * n_rows, cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaMemcpyAsync(hp.data(), S.ptr, sizeof(int64_t) * nptr, cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    dfree(d_flag);
  }
  int h_err = 0;
  PSC_CUDA(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(d_err);
  PSC_REQUIRE(h_err == 0, PSC_ERR_STATE,
              h_err == 2 ? "DIA slice fill mismatch" : "column not in the owned block nor in the assembled halo");
  std::vector<int32_t> in, bd;
  S.nnz_ell = sell ? 0 : nnz;
  for (int64_t u = 0; u < nu; ++u) {
    int f = 0;
    if (sell) {
      f = flag[u];
      S.max_width = std::max<int>(S.max_width, (int)((hp[u + 1] - hp[u]) / 32));
      if (hdia[u]) S.n_dia++;
      else S.nnz_ell += hsnnz[u];
    } else {
      for (int64_t i = u * RU; i < std::min<int64_t>(n_rows, (u + 1) * RU); ++i) {
        f |= flag[i];
        S.max_width = std::max<int>(S.max_width, (int)(hp[i + 1] - hp[i]));
      }
      if (u % 8 == 0) {
        const int64_t r1 = std::min<int64_t>(n_rows, (u + 8) * RU);
        S.max_chunk = std::max<int64_t>(S.max_chunk, hp[r1] - hp[u * RU]);
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
  dfree(S.cptr);
  dfree(S.hdr);
  dfree(S.col);
  dfree(S.val);
  dfree(S.interior);
  dfree(S.boundary);
  dfree(S.perm);
  dfree(S.iperm);
  dfree(S.slot);
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

namespace psc {
__global__ void scatter_values_kernel(int64_t nnz, const int64_t* __restrict__ slot, const double* __restrict__ v,
                                      double* __restrict__ val) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) val[slot[k]] = v[k];
}
void sell_update_values(psc_ctx* ctx, Sell& S, const double* d_newval, cudaStream_t s) {
  if (S.nnz == 0) return;
  scatter_values_kernel<<<(unsigned)((S.nnz + 255) / 256), 256, 0, s>>>(S.nnz, S.slot, d_newval, S.val);
  PSC_CUDA(cudaGetLastError());
  ctx->launches++;
}
}  // namespace psc
