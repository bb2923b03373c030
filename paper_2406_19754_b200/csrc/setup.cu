// setup.cu — the AMG set-up on the device: decoupled
// Vanek-Mandel-Brezina aggregation, the tentative prolongator of
// Eq. (3) with w = 1, its smoothing P = (I - omega D^-1 A) P^ with
// omega = 1/||D^-1 A||_inf, R = P^T and the Galerkin product
// A_{l+1} = P^T A P — the part the paper names as still "executed
// mostly on the CPU side" and as future work.
//
// Readings: R17 theta, R18 phases, R19 stop rule, R21 omega, R26
// phase 1 = the greedy VMB root rule visited in increasing index.  Phase 1 is that
// greedy rule's fixed point computed in parallel rounds: an undecided node becomes a
// root when it is the smallest undecided index within two strong edges and no root
// is within two strong edges; nodes with a root within two strong edges drop out.
// A node is decided only after every smaller index within two strong edges, so the
// roots equal those of the sequential sweep in increasing index.
//
// Every floating-point result is computed in the order the definitions state (row
// sums in column order, the Galerkin products k -> K row by row) with one rounding per
// operation and no FMA contraction (__dmul_rn / __dadd_rn), so the set-up is
// reproducible bit for bit by a plain sequential implementation.  One rank.
#include <cub/cub.cuh>

#include <chrono>
#include <memory>
#include <climits>
#include <cstdio>
#include <cstring>

#include "kernels.h"

namespace psc {
namespace {

constexpr int kT = 256;

struct DCsr {  // device CSR, int64 row offsets and columns
  int64_t n = 0, ncols = 0, nnz = 0;
  int64_t* ptr = nullptr;
  int64_t* col = nullptr;
  double* val = nullptr;
};
void dcsr_free(DCsr& m) {
  dfree(m.ptr);
  dfree(m.col);
  dfree(m.val);
  m = DCsr();
}

unsigned blocks(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + kT - 1) / kT); }

int64_t d2h_i64(const int64_t* p, cudaStream_t s) {
  int64_t v = 0;
  PSC_CUDA(cudaMemcpyAsync(&v, p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  PSC_CUDA(cudaStreamSynchronize(s));
  return v;
}

// exclusive scan of cnt[0..n) into out[0..n], out[n] = total; returns the total
int64_t scan(const int64_t* cnt, int64_t* out, int64_t n, cudaStream_t s) {
  PSC_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
  if (n > 0) {
    size_t tb = 0;
    PSC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, out + 1, n, s));
    void* tmp = dalloc<char>(tb);
    PSC_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, cnt, out + 1, n, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    dfree(tmp);
  }
  return d2h_i64(out + n, s);
}

// ------------------------------------------------------------ strength + diag
__global__ void diag_kernel(DCsr A, double* __restrict__ d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  double v = 0.0;
  for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
    if (A.col[k] == i) v = A.val[k];
  d[i] = v;
}

// N_i(theta) of P:215-216: j != i, |a_ij| >= theta sqrt(a_ii a_jj)
__global__ void strong_kernel(DCsr A, const double* __restrict__ d, double theta, uint8_t* __restrict__ st) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
    const int64_t j = A.col[k];
    st[k] = (j != i && fabs(A.val[k]) >= __dmul_rn(theta, __dsqrt_rn(__dmul_rn(d[i], d[j])))) ? 1 : 0;
  }
}

// ------------------------------------------------------------ phase 1 rounds
enum : int8_t { kUndecided = 0, kRoot = 1, kOut = 2 };

// m1[i] = smallest undecided index in {i} u N_i; r1[i] = a root in {i} u N_i
__global__ void mis_a_kernel(DCsr A, const uint8_t* __restrict__ st, const int8_t* __restrict__ state,
                             int64_t* __restrict__ m1, uint8_t* __restrict__ r1) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  int64_t m = state[i] == kUndecided ? i : LLONG_MAX;
  uint8_t r = state[i] == kRoot;
  for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
    if (!st[k]) continue;
    const int64_t j = A.col[k];
    const int8_t sj = state[j];
    if (sj == kUndecided && j < m) m = j;
    r |= (sj == kRoot);
  }
  m1[i] = m;
  r1[i] = r;
}

// undecided i: a root within two strong edges -> out; else the smallest undecided
// index within two strong edges is i -> root
__global__ void mis_b_kernel(DCsr A, const uint8_t* __restrict__ st, int8_t* __restrict__ state,
                             const int64_t* __restrict__ m1, const uint8_t* __restrict__ r1,
                             unsigned long long* __restrict__ undecided) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n || state[i] != kUndecided) return;
  int64_t m = m1[i];
  bool r = r1[i];
  for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
    if (!st[k]) continue;
    const int64_t j = A.col[k];
    if (m1[j] < m) m = m1[j];
    r |= r1[j] != 0;
  }
  if (r) state[i] = kOut;
  else if (m == i) state[i] = kRoot;
  else atomicAdd(undecided, 1ull);
}

__global__ void root_flag_kernel(int64_t n, const int8_t* __restrict__ state, int64_t* __restrict__ f) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = state[i] == kRoot;
}

// phase 1 membership: a root's aggregate is the root and its strong neighbours
__global__ void phase1_kernel(DCsr A, const uint8_t* __restrict__ st, const int8_t* __restrict__ state,
                              const int64_t* __restrict__ rid, int64_t* __restrict__ agg1) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  int64_t a = -1;
  if (state[i] == kRoot) {
    a = rid[i];
  } else {
    for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
      if (st[k] && state[A.col[k]] == kRoot) a = rid[A.col[k]];  // at most one (roots >= 3 apart)
  }
  agg1[i] = a;
}

// phase 2 (R18): join the phase-1 aggregate of the strongest strong
// neighbour (|a_ij| / sqrt(a_ii a_jj)), ties to the lowest id
__global__ void phase2_kernel(DCsr A, const uint8_t* __restrict__ st, const double* __restrict__ d,
                              const int64_t* __restrict__ agg1, int64_t* __restrict__ agg,
                              unsigned long long* __restrict__ left) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  if (agg1[i] >= 0) {
    agg[i] = agg1[i];
    return;
  }
  double best = -1.0;
  int64_t ba = -1;
  for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
    const int64_t j = A.col[k];
    if (!st[k] || agg1[j] < 0) continue;
    const double s = __ddiv_rn(fabs(A.val[k]), __dsqrt_rn(__dmul_rn(d[i], d[j])));
    const int64_t a = agg1[j];
    if (s > best || (s == best && a < ba)) {
      best = s;
      ba = a;
    }
  }
  agg[i] = ba;
  if (ba < 0) atomicAdd(left, 1ull);
}

// ------------------------------------------------------------ omega
// t_i = sum_j |a_ij| / |a_ii| (column order); omega = 1 / max_i t_i.  Non-negative
// doubles order like their bit patterns, so an integer atomicMax is exact.
__global__ void rowscale_kernel(DCsr A, unsigned long long* __restrict__ mx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  double s = 0.0, dii = 0.0;
  for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
    s = __dadd_rn(s, fabs(A.val[k]));
    if (A.col[k] == i) dii = A.val[k];
  }
  const double t = __ddiv_rn(s, fabs(dii));
  atomicMax(mx, (unsigned long long)__double_as_longlong(t));
}

// ------------------------------------------------------------ smoothed prolongator
// Row i of P = (I - omega D^-1 A) P^: distinct
// aggregates J of row i's columns in order of first appearance, t_J summed in
// column order, in a scratch slice of row i's own length; then
// P_iJ = 1 - s t_J (J = agg(i)) or -s t_J, s = omega / a_ii, columns increasing.
__global__ void prol_kernel(DCsr A, const int64_t* __restrict__ agg, double omega, int64_t* __restrict__ sJ,
                            double* __restrict__ sT, int64_t* __restrict__ cnt, const int64_t* __restrict__ pptr,
                            int64_t* __restrict__ pcol, double* __restrict__ pval) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  const int64_t b = A.ptr[i];
  int64_t o = b;
  double dii = 0.0;
  for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
    if (A.col[k] == i) dii = A.val[k];
    const int64_t J = agg[A.col[k]];
    int64_t t = b;
    while (t < o && sJ[t] != J) ++t;
    if (t == o) {
      sJ[o] = J;
      sT[o] = A.val[k];
      ++o;
    } else {
      sT[t] = __dadd_rn(sT[t], A.val[k]);
    }
  }
  if (!pptr) {  // counting pass
    cnt[i] = o - b;
    return;
  }
  const double s = __ddiv_rn(omega, dii);
  const int64_t q0 = pptr[i];
  const int64_t ai = agg[i];
  for (int64_t t = b; t < o; ++t) {  // insertion into the output row by increasing J
    const int64_t J = sJ[t];
    const double v = __dmul_rn(s, sT[t]);
    const double pv = (J == ai) ? __dsub_rn(1.0, v) : -v;
    int64_t y = q0 + (t - b) - 1;
    while (y >= q0 && pcol[y] > J) {
      pcol[y + 1] = pcol[y];
      pval[y + 1] = pval[y];
      --y;
    }
    pcol[y + 1] = J;
    pval[y + 1] = pv;
  }
}

// ------------------------------------------------------------ transpose
__global__ void colcount_kernel(DCsr P, int64_t* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  for (int64_t k = P.ptr[i]; k < P.ptr[i + 1]; ++k) atomicAdd((unsigned long long*)&cnt[P.col[k]], 1ull);
}
__global__ void tfill_kernel(DCsr P, int64_t* __restrict__ fill, int64_t* __restrict__ rcol,
                             double* __restrict__ rval) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  for (int64_t k = P.ptr[i]; k < P.ptr[i + 1]; ++k) {
    const int64_t o = (int64_t)atomicAdd((unsigned long long*)&fill[P.col[k]], 1ull);
    rcol[o] = i;
    rval[o] = P.val[k];
  }
}
// rows of R by increasing column (the slot order above depends on timing)
__global__ void rowsort_kernel(DCsr M) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M.n) return;
  const int64_t b = M.ptr[r], e = M.ptr[r + 1];
  for (int64_t x = b + 1; x < e; ++x) {
    const int64_t c = M.col[x];
    const double v = M.val[x];
    int64_t y = x - 1;
    while (y >= b && M.col[y] > c) {
      M.col[y + 1] = M.col[y];
      M.val[y + 1] = M.val[y];
      --y;
    }
    M.col[y + 1] = c;
    M.val[y + 1] = v;
  }
}

// ------------------------------------------------------------ Galerkin R A P
__device__ __forceinline__ uint32_t hslot(int64_t K, uint32_t mask) {
  return (uint32_t)(((uint64_t)K * 0x9E3779B97F4A7C15ull) >> 32) & mask;
}

__global__ void mark_kernel(int64_t n, const int64_t* __restrict__ rows, int64_t* __restrict__ cnt) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) cnt[rows[q]] = -1;
}
double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

// ------------------------------------------------------------ one level
struct AmgLevel {
  DCsr A, P, R;        // P, R absent at the coarsest level
  int64_t* agg = nullptr;  // n: aggregate of each node
  int8_t* root = nullptr;  // n
  double omega = 0.0;
  int mis_rounds = 0;
};

}  // namespace psc

struct psc_amg_s {
  psc_ctx* ctx = nullptr;
  psc_amg_opts opt{};
  std::vector<psc::AmgLevel> lv;
  double t_aggregate = 0.0, t_prolongator = 0.0, t_transpose = 0.0, t_galerkin = 0.0, t_total = 0.0;
  // objects created by psc_amg_hier_create (owned here)
  std::vector<psc_desc*> descs;
  std::vector<psc_mat*> mats;
};

namespace psc {
namespace {

// decoupled VMB aggregation of one level (one rank): returns the number of aggregates
int64_t aggregate(psc_ctx* ctx, AmgLevel& L, double theta) {
  NvtxRange nv("psc_amg_aggregate");
  cudaStream_t s = ctx->stream;
  const DCsr& A = L.A;
  const int64_t n = A.n;
  double* d = dalloc<double>(n);
  uint8_t* st = dalloc<uint8_t>(A.nnz);
  int8_t* state = dalloc<int8_t>(n);
  int64_t* m1 = dalloc<int64_t>(n);
  uint8_t* r1 = dalloc<uint8_t>(n);
  unsigned long long* ctr = dalloc<unsigned long long>(1);
  diag_kernel<<<blocks(n), kT, 0, s>>>(A, d);
  strong_kernel<<<blocks(n), kT, 0, s>>>(A, d, theta, st);
  PSC_CUDA(cudaMemsetAsync(state, kUndecided, n, s));
  PSC_CUDA(cudaGetLastError());
  // rounds until every node is decided (the count is read back every 8 rounds)
  for (int round = 0;; ++round) {
    PSC_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s));
    mis_a_kernel<<<blocks(n), kT, 0, s>>>(A, st, state, m1, r1);
    mis_b_kernel<<<blocks(n), kT, 0, s>>>(A, st, state, m1, r1, ctr);
    L.mis_rounds = round + 1;
    if ((round & 7) == 7 || n < 4096) {
      unsigned long long left = 0;
      PSC_CUDA(cudaMemcpyAsync(&left, ctr, sizeof(left), cudaMemcpyDeviceToHost, s));
      PSC_CUDA(cudaStreamSynchronize(s));
      if (left == 0) break;
    }
    PSC_REQUIRE(round < 4 * n + 64, PSC_ERR_STATE, "VMB phase 1 did not converge");
  }
  int64_t* f = dalloc<int64_t>(n);
  int64_t* rid = dalloc<int64_t>(n + 1);
  root_flag_kernel<<<blocks(n), kT, 0, s>>>(n, state, f);
  const int64_t nc = scan(f, rid, n, s);
  int64_t* agg1 = f;  // reuse
  phase1_kernel<<<blocks(n), kT, 0, s>>>(A, st, state, rid, agg1);
  L.agg = dalloc<int64_t>(n);
  PSC_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s));
  phase2_kernel<<<blocks(n), kT, 0, s>>>(A, st, d, agg1, L.agg, ctr);
  PSC_CUDA(cudaGetLastError());
  unsigned long long left = 0;
  PSC_CUDA(cudaMemcpyAsync(&left, ctr, sizeof(left), cudaMemcpyDeviceToHost, s));
  L.root = state;  // kRoot marks the roots
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(d);
  dfree(st);
  dfree(m1);
  dfree(r1);
  dfree(ctr);
  dfree(f);
  dfree(rid);
  PSC_REQUIRE(left == 0, PSC_ERR_STATE, "VMB phase 3 reached (node farther than two strong edges from every root)");
  return nc;
}

double omega_of(psc_ctx* ctx, const DCsr& A) {
  cudaStream_t s = ctx->stream;
  unsigned long long* mx = dalloc<unsigned long long>(1);
  PSC_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), s));
  rowscale_kernel<<<blocks(A.n), kT, 0, s>>>(A, mx);
  PSC_CUDA(cudaGetLastError());
  unsigned long long v = 0;
  PSC_CUDA(cudaMemcpyAsync(&v, mx, sizeof(v), cudaMemcpyDeviceToHost, s));
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(mx);
  double m;
  std::memcpy(&m, &v, sizeof(m));
  return 1.0 / m;
}

DCsr prolongator(psc_ctx* ctx, const AmgLevel& L, int64_t nc) {
  cudaStream_t s = ctx->stream;
  const DCsr& A = L.A;
  int64_t* sJ = dalloc<int64_t>(A.nnz);
  double* sT = dalloc<double>(A.nnz);
  int64_t* cnt = dalloc<int64_t>(A.n);
  DCsr P;
  P.n = A.n;
  P.ncols = nc;
  P.ptr = dalloc<int64_t>(A.n + 1);
  prol_kernel<<<blocks(A.n), kT, 0, s>>>(A, L.agg, L.omega, sJ, sT, cnt, nullptr, nullptr, nullptr);
  PSC_CUDA(cudaGetLastError());
  P.nnz = scan(cnt, P.ptr, A.n, s);
  P.col = dalloc<int64_t>(P.nnz);
  P.val = dalloc<double>(P.nnz);
  prol_kernel<<<blocks(A.n), kT, 0, s>>>(A, L.agg, L.omega, sJ, sT, cnt, P.ptr, P.col, P.val);
  PSC_CUDA(cudaGetLastError());
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(sJ);
  dfree(sT);
  dfree(cnt);
  return P;
}

DCsr transpose(psc_ctx* ctx, const DCsr& P) {
  cudaStream_t s = ctx->stream;
  DCsr R;
  R.n = P.ncols;
  R.ncols = P.n;
  R.nnz = P.nnz;
  int64_t* cnt = dalloc<int64_t>(R.n);
  PSC_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * R.n, s));
  colcount_kernel<<<blocks(P.n), kT, 0, s>>>(P, cnt);
  R.ptr = dalloc<int64_t>(R.n + 1);
  scan(cnt, R.ptr, R.n, s);
  PSC_CUDA(cudaMemcpyAsync(cnt, R.ptr, sizeof(int64_t) * R.n, cudaMemcpyDeviceToDevice, s));
  R.col = dalloc<int64_t>(R.nnz);
  R.val = dalloc<double>(R.nnz);
  tfill_kernel<<<blocks(P.n), kT, 0, s>>>(P, cnt, R.col, R.val);
  rowsort_kernel<<<blocks(R.n), kT, 0, s>>>(R);
  PSC_CUDA(cudaGetLastError());
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(cnt);
  return R;
}

// ------------------------------------------------------------ sparse products
// Z = X Y row by row (Gustavson), every Z[i, K] accumulated exactly in the order of
// the definition (k along X's row i, then K along Y's row k; acc = acc + x y with one
// rounding per operation, no FMA), so the result is bit-identical to a sequential
// implementation.  A row is first tried in a small per-thread table; the rows that do
// not fit go to one warp per row with a larger table (shared, then global memory).
// Every stage has a count pass (cnt[i] = distinct K, or -1: redo at the next stage)
// and a fill pass (columns increasing) over the rows it holds.

// stage 0: thread per row, kSmallT-slot open-addressing table in shared memory (32-bit
// keys: K < 2^31 on one rank), interleaved [slot][thread] so that the threads of a warp
// probing the same slot index hit different banks
constexpr int kSmallT = 64;
constexpr int kProdThreads = 128;
constexpr int kProdSmem = kProdThreads * kSmallT * (4 + 8 + 1);
__global__ void __launch_bounds__(kProdThreads) prod_thread_kernel(DCsr X, DCsr Y, int64_t* __restrict__ cnt,
                                                                   const int64_t* __restrict__ cptr,
                                                                   int64_t* __restrict__ ccol,
                                                                   double* __restrict__ cval) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* acc = reinterpret_cast<double*>(sm);
  int32_t* key = reinterpret_cast<int32_t*>(sm + kProdThreads * kSmallT * 8);
  uint8_t* tl = sm + kProdThreads * kSmallT * 12;
  const int t = threadIdx.x;
  constexpr int cap = kSmallT - kSmallT / 4;
  for (int h = 0; h < kSmallT; ++h) key[h * kProdThreads + t] = -1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + t; i < X.n; i += (int64_t)gridDim.x * blockDim.x) {
    if (cptr && cnt[i] < 0) continue;
    int nt = 0;
    bool over = false;
    for (int64_t b = X.ptr[i]; b < X.ptr[i + 1] && !over; ++b) {
      const int64_t k = X.col[b];
      const double xv = X.val[b];
      for (int64_t c = Y.ptr[k]; c < Y.ptr[k + 1]; ++c) {
        const int32_t K = (int32_t)Y.col[c];
        uint32_t h = hslot(K, kSmallT - 1);
        while (key[h * kProdThreads + t] != -1 && key[h * kProdThreads + t] != K) h = (h + 1) & (kSmallT - 1);
        const int s = h * kProdThreads + t;
        if (key[s] == -1) {
          if (nt == cap) {
            over = true;
            break;
          }
          key[s] = K;
          acc[s] = 0.0;
          tl[nt * kProdThreads + t] = (uint8_t)h;
          ++nt;
        }
        acc[s] = __dadd_rn(acc[s], __dmul_rn(xv, Y.val[c]));
      }
    }
    if (!cptr) {
      cnt[i] = over ? -1 : nt;
    } else {
      const int64_t q0 = cptr[i];
      for (int x = 0; x < nt; ++x) {  // insertion by increasing K
        const int s = tl[x * kProdThreads + t] * kProdThreads + t;
        const int64_t K = key[s];
        const double v = acc[s];
        int64_t y = q0 + x - 1;
        while (y >= q0 && ccol[y] > K) {
          ccol[y + 1] = ccol[y];
          cval[y + 1] = cval[y];
          --y;
        }
        ccol[y + 1] = K;
        cval[y + 1] = v;
      }
    }
    for (int x = 0; x < nt; ++x) key[tl[x * kProdThreads + t] * kProdThreads + t] = -1;
  }
}

// stages >= 1: one warp per row.  The warp walks X's row i in order and spreads each
// Y row k over its lanes: the K of one Y row are distinct, so every acc[K] still
// receives its terms in the sequential order.  The table (T slots, keys / values,
// plus the compaction list used by the fill pass) is in shared memory (T = kWT) or in
// a per-warp slice of global memory (larger T).
constexpr int kWT = 1024;
constexpr int kWCap = 768;
constexpr int kProdWarps = 4;
constexpr int kProdWarpSmem = kProdWarps * kWT * (4 + 8 + 4 + 8);
struct WarpTab {
  int32_t* key;
  double* val;
  int32_t* lk;
  double* lv;
};
__global__ void __launch_bounds__(kProdWarps * 32) prod_warp_kernel(DCsr X, DCsr Y, int64_t* __restrict__ cnt,
                                                                    const int64_t* __restrict__ rows, int64_t nrows,
                                                                    int T, int wcap, unsigned char* gtab,
                                                                    const int64_t* __restrict__ cptr,
                                                                    int64_t* __restrict__ ccol,
                                                                    double* __restrict__ cval) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int tcnt[kProdWarps];
  constexpr unsigned kFull = 0xffffffffu;
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kProdWarps + wi;
  unsigned char* base = gtab ? gtab + (size_t)gw * T * 24 : sm + (size_t)wi * T * 24;
  WarpTab tb{reinterpret_cast<int32_t*>(base), reinterpret_cast<double*>(base + (size_t)T * 4),
             reinterpret_cast<int32_t*>(base + (size_t)T * 12), reinterpret_cast<double*>(base + (size_t)T * 16)};
  volatile int32_t* vkey = tb.key;
  volatile int* vcnt = &tcnt[wi];
  const uint32_t mask = (uint32_t)T - 1;
  for (int h = lane; h < T; h += 32) tb.key[h] = -1;
  if (lane == 0) tcnt[wi] = 0;
  __syncwarp();
  const int64_t nw = (int64_t)gridDim.x * kProdWarps;
  for (int64_t q = gw; q < nrows; q += nw) {
    const int64_t i = rows ? rows[q] : q;
    if (cptr && cnt[i] < 0) continue;
    bool over = false;
    const int64_t b1 = X.ptr[i + 1];
    for (int64_t bb = X.ptr[i]; bb < b1 && !over; bb += 32) {
      // lane j holds (x, Y row range) of entry bb + j of X's row
      int64_t pb = 0, pe = 0;
      double xl = 0.0;
      if (bb + lane < b1) {
        const int64_t k = X.col[bb + lane];
        xl = X.val[bb + lane];
        pb = Y.ptr[k];
        pe = Y.ptr[k + 1];
      }
      const int np = (int)(b1 - bb < 32 ? b1 - bb : 32);
      for (int j = 0; j < np && !over; ++j) {
        const int64_t cb = __shfl_sync(kFull, pb, j);
        const int64_t ce = __shfl_sync(kFull, pe, j);
        const double xv = __shfl_sync(kFull, xl, j);
        for (int64_t c0 = cb; c0 < ce; c0 += 32) {
          const int64_t c = c0 + lane;
          if (c < ce) {
            const int32_t K = (int32_t)Y.col[c];
            const double v = __dmul_rn(xv, Y.val[c]);
            uint32_t h = hslot(K, mask);
            for (;;) {
              int32_t cur = vkey[h];
              if (cur == -1) {
                cur = atomicCAS(&tb.key[h], -1, K);
                if (cur == -1) {
                  atomicAdd(&tcnt[wi], 1);
                  tb.val[h] = 0.0;
                  break;
                }
              }
              if (cur == K) break;
              h = (h + 1) & mask;
            }
            tb.val[h] = __dadd_rn(tb.val[h], v);
          }
          __syncwarp();
          // at most 32 inserts per step: a table past wcap (<= 3/4 T) still has room
          if (*vcnt > wcap) {
            over = true;
            break;
          }
        }
      }
    }
    __syncwarp();
    if (!cptr) {
      if (lane == 0) cnt[i] = over ? -1 : *vcnt;
    } else {
      // compact the occupied slots, then place each by its rank among the keys
      int nt = 0;
      for (int b = 0; b < T; b += 32) {
        const int32_t K = tb.key[b + lane];
        const unsigned m = __ballot_sync(kFull, K != -1);
        if (K != -1) {
          const int pos = nt + __popc(m & ((1u << lane) - 1u));
          tb.lk[pos] = K;
          tb.lv[pos] = tb.val[b + lane];
        }
        nt += __popc(m);
      }
      __syncwarp();
      const int64_t q0 = cptr[i];
      for (int x = lane; x < nt; x += 32) {
        const int32_t K = tb.lk[x];
        int rank = 0;
        for (int y = 0; y < nt; ++y) rank += tb.lk[y] < K;
        ccol[q0 + rank] = K;
        cval[q0 + rank] = tb.lv[x];
      }
    }
    __syncwarp();
    for (int h = lane; h < T; h += 32) tb.key[h] = -1;
    if (lane == 0) tcnt[wi] = 0;
    __syncwarp();
  }
}

// one escalation stage of the warp kernel: table size, the rows it holds, and (global
// stages) the per-warp tables
struct ProdStage {
  int T = 0;
  int64_t* rows = nullptr;
  int64_t nrows = 0;
  unsigned char* gtab = nullptr;
  unsigned grid = 1;
};

// PSC_RAP_WCAP lowers the shared-memory warp stage's row capacity (tests: reach the
// global stages on small problems)
int warp_cap() {
  const char* e = getenv("PSC_RAP_WCAP");
  const int v = e ? atoi(e) : kWCap;
  return v >= 1 && v <= kWCap ? v : kWCap;
}

void prod_thread_launch(psc_ctx* ctx, const DCsr& X, const DCsr& Y, int64_t* cnt, const int64_t* cptr,
                        int64_t* ccol, double* cval, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    PSC_CUDA(cudaFuncSetAttribute(prod_thread_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kProdSmem));
    attr = true;
  }
  const int64_t need = (X.n + kProdThreads - 1) / kProdThreads;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)ctx->num_sms * 2));
  prod_thread_kernel<<<grid, kProdThreads, kProdSmem, s>>>(X, Y, cnt, cptr, ccol, cval);
  PSC_CUDA(cudaGetLastError());
}

void prod_warp_launch(const DCsr& X, const DCsr& Y, int64_t* cnt, const ProdStage& st, const int64_t* cptr,
                      int64_t* ccol, double* cval, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    PSC_CUDA(cudaFuncSetAttribute(prod_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kProdWarpSmem));
    attr = true;
  }
  const int wcap = st.gtab ? st.T - st.T / 4 : warp_cap();
  prod_warp_kernel<<<st.grid, kProdWarps * 32, st.gtab ? 0 : kProdWarpSmem, s>>>(X, Y, cnt, st.rows, st.nrows, st.T,
                                                                                wcap, st.gtab, cptr, ccol, cval);
  PSC_CUDA(cudaGetLastError());
}

// Z = X Y (X.n rows, Y.ncols columns, columns increasing per row)
DCsr spgemm(psc_ctx* ctx, const DCsr& X, const DCsr& Y) {
  cudaStream_t s = ctx->stream;
  const int64_t n = X.n;
  PSC_REQUIRE(Y.ncols < INT32_MAX, PSC_ERR_STATE, "sparse product: more than 2^31 columns");
  int64_t* cnt = dalloc<int64_t>(std::max<int64_t>(n, 1));
  prod_thread_launch(ctx, X, Y, cnt, nullptr, nullptr, nullptr, s);
  std::vector<ProdStage> stages;
  std::vector<int64_t> hc(n);
  for (;;) {
    if (n) PSC_CUDA(cudaMemcpyAsync(hc.data(), cnt, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> big;
    for (int64_t i = 0; i < n; ++i)
      if (hc[i] < 0) big.push_back(i);
    if (big.empty()) break;
    ProdStage st;
    st.T = stages.empty() ? kWT : (stages.size() == 1 ? 8192 : stages.back().T * 8);
    PSC_REQUIRE(st.T <= (1 << 30) && st.T <= 4 * Y.ncols + 8192, PSC_ERR_STATE, "sparse product: row too long");
    st.nrows = (int64_t)big.size();
    st.rows = dalloc<int64_t>(big.size());
    PSC_CUDA(cudaMemcpyAsync(st.rows, big.data(), sizeof(int64_t) * big.size(), cudaMemcpyHostToDevice, s));
    int64_t nwarps = std::min<int64_t>(st.nrows, (int64_t)ctx->num_sms * 16);
    if (!stages.empty()) {  // global tables: at most ~1.5 GB of them
      nwarps = std::min<int64_t>(nwarps, std::max<int64_t>(kProdWarps, ((int64_t)3 << 29) / (24 * (int64_t)st.T)));
      nwarps = (nwarps + kProdWarps - 1) / kProdWarps * kProdWarps;
      st.gtab = dalloc<unsigned char>((size_t)nwarps * st.T * 24);  // keys cleared by the kernel
    }
    st.grid = (unsigned)std::max<int64_t>(1, (nwarps + kProdWarps - 1) / kProdWarps);
    prod_warp_launch(X, Y, cnt, st, nullptr, nullptr, nullptr, s);
    stages.push_back(st);
  }
  DCsr Z;
  Z.n = n;
  Z.ncols = Y.ncols;
  Z.ptr = dalloc<int64_t>(n + 1);
  Z.nnz = scan(cnt, Z.ptr, n, s);
  Z.col = dalloc<int64_t>(std::max<int64_t>(Z.nnz, 1));
  Z.val = dalloc<double>(std::max<int64_t>(Z.nnz, 1));
  // fill: each row by the stage whose table held it (the others skip it: cnt < 0)
  for (size_t q = 0; q <= stages.size(); ++q) {
    // rows escalated past stage q (the lists are nested, so marking every later list
    // marks exactly them) are skipped; stage q does the rest of its rows
    PSC_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * n, s));
    for (size_t r = q; r < stages.size(); ++r)
      mark_kernel<<<blocks(stages[r].nrows), kT, 0, s>>>(stages[r].nrows, stages[r].rows, cnt);
    if (q == 0) prod_thread_launch(ctx, X, Y, cnt, Z.ptr, Z.col, Z.val, s);
    else prod_warp_launch(X, Y, cnt, stages[q - 1], Z.ptr, Z.col, Z.val, s);
    PSC_CUDA(cudaGetLastError());
  }
  PSC_CUDA(cudaStreamSynchronize(s));
  for (auto& st : stages) {
    dfree(st.rows);
    dfree(st.gtab);
  }
  dfree(cnt);
  return Z;
}

// Galerkin A_c = R A P, reading R31: R (A P), two sparse products.
DCsr galerkin(psc_ctx* ctx, const DCsr& R, const DCsr& A, const DCsr& P) {
  NvtxRange nv("psc_amg_galerkin");
  DCsr AP = spgemm(ctx, A, P);
  DCsr C = spgemm(ctx, R, AP);
  dcsr_free(AP);
  return C;
}

void amg_free(psc_amg* a) {
  for (auto& L : a->lv) {
    dcsr_free(L.A);
    dcsr_free(L.P);
    dcsr_free(L.R);
    dfree(L.agg);
    dfree(L.root);
  }
  a->lv.clear();
}

}  // namespace
}  // namespace psc

using namespace psc;

extern "C" {

int psc_amg_build(psc_ctx* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                  const psc_amg_opts* opts, psc_amg** out) {
  psc_amg* a = nullptr;
  try {
    PSC_REQUIRE(ctx && out && row_ptr && n >= 1, PSC_ERR_ARG, "bad argument");
    PSC_REQUIRE(ctx->nranks == 1, PSC_ERR_STATE, "psc_amg_build: one rank only (the decoupled multi-rank set-up "
                                                 "is built by the caller and given to psc_hier_create)");
    PSC_REQUIRE(row_ptr[0] == 0, PSC_ERR_ARG, "row_ptr[0] != 0");
    for (int64_t i = 0; i < n; ++i) {
      PSC_REQUIRE(row_ptr[i + 1] >= row_ptr[i], PSC_ERR_ARG, "row_ptr decreasing");
      bool diag = false;
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        PSC_REQUIRE(col[k] >= 0 && col[k] < n && (k == row_ptr[i] || col[k] > col[k - 1]), PSC_ERR_ARG,
                    "columns must be strictly increasing within a row and in [0, n)");
        if (col[k] == i) diag = val[k] > 0.0;
      }
      PSC_REQUIRE(diag, PSC_ERR_ARG, "every row needs a positive diagonal (N_i(theta), P:215-216)");
    }
    psc_amg_opts o = opts ? *opts : psc_amg_opts{0.01, 20, 200, 0.75};
    PSC_REQUIRE(o.theta >= 0.0 && o.theta < 1.0 && o.max_levels >= 1 && o.coarse_target >= 1 &&
                    o.stall_ratio > 0.0 && o.stall_ratio <= 1.0,
                PSC_ERR_ARG, "bad psc_amg_opts");
    PSC_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    a = new psc_amg_s();
    a->ctx = ctx;
    a->opt = o;
    const auto t0 = std::chrono::steady_clock::now();
    AmgLevel L0;
    const int64_t nnz = row_ptr[n];
    L0.A.n = L0.A.ncols = n;
    L0.A.nnz = nnz;
    L0.A.ptr = dalloc<int64_t>(n + 1);
    L0.A.col = dalloc<int64_t>(nnz);
    L0.A.val = dalloc<double>(nnz);
    PSC_CUDA(cudaMemcpyAsync(L0.A.ptr, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    PSC_CUDA(cudaMemcpyAsync(L0.A.col, col, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, s));
    PSC_CUDA(cudaMemcpyAsync(L0.A.val, val, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    a->lv.push_back(L0);
    for (;;) {
      AmgLevel& L = a->lv.back();
      if (L.A.n <= o.coarse_target || (int)a->lv.size() >= o.max_levels) break;
      auto t = std::chrono::steady_clock::now();
      const int64_t nc = aggregate(ctx, L, o.theta);
      a->t_aggregate += secs_since(t);
      if ((double)nc > o.stall_ratio * (double)L.A.n || nc >= L.A.n) {  // R19: coarsening stalls
        dfree(L.agg);
        dfree(L.root);
        L.agg = nullptr;
        L.root = nullptr;
        break;
      }
      t = std::chrono::steady_clock::now();
      L.omega = omega_of(ctx, L.A);
      L.P = prolongator(ctx, L, nc);
      a->t_prolongator += secs_since(t);
      t = std::chrono::steady_clock::now();
      L.R = transpose(ctx, L.P);
      a->t_transpose += secs_since(t);
      t = std::chrono::steady_clock::now();
      AmgLevel N;
      N.A = galerkin(ctx, L.R, L.A, L.P);
      a->t_galerkin += secs_since(t);
      if (getenv("PSC_AMG_VERBOSE"))
        fprintf(stderr, "[psc_amg] level %d: n %lld nnz %lld -> %lld rows, %lld nnz; rounds %d, galerkin %.3f s\n",
                (int)a->lv.size() - 1, (long long)L.A.n, (long long)L.A.nnz, (long long)N.A.n, (long long)N.A.nnz,
                L.mis_rounds, secs_since(t));
      a->lv.push_back(N);
    }
    a->t_total = secs_since(t0);
    *out = a;
    return PSC_OK;
  } catch (const Error& e) {
    if (a) {
      amg_free(a);
      delete a;
    }
    if (ctx) ctx->err = e.what();
    return e.code;
  }
}

int psc_amg_info(psc_amg* a, int* nlevels, int64_t* n, int64_t* nnz_A, int64_t* nnz_P, double* omega,
                 int* mis_rounds, double* seconds) {
  if (!a || !nlevels) return PSC_ERR_ARG;
  const int L = (int)a->lv.size();
  *nlevels = L;
  for (int l = 0; l < L; ++l) {
    if (n) n[l] = a->lv[l].A.n;
    if (nnz_A) nnz_A[l] = a->lv[l].A.nnz;
    if (nnz_P) nnz_P[l] = a->lv[l].P.nnz;
    if (omega) omega[l] = a->lv[l].omega;
    if (mis_rounds) mis_rounds[l] = a->lv[l].mis_rounds;
  }
  if (seconds) {
    seconds[0] = a->t_aggregate;
    seconds[1] = a->t_prolongator;
    seconds[2] = a->t_transpose;
    seconds[3] = a->t_galerkin;
    seconds[4] = a->t_total;
  }
  return PSC_OK;
}

int psc_amg_level_csr(psc_amg* a, int level, int kind, int64_t* row_ptr, int64_t* col, double* val) {
  psc_ctx* ctx = a ? a->ctx : nullptr;
  try {
    PSC_REQUIRE(a && level >= 0 && level < (int)a->lv.size() && kind >= 0 && kind <= 2, PSC_ERR_ARG, "bad argument");
    const AmgLevel& L = a->lv[level];
    const DCsr& M = kind == 0 ? L.A : (kind == 1 ? L.P : L.R);
    PSC_REQUIRE(M.ptr, PSC_ERR_STATE, "no such matrix at this level (P/R absent at the coarsest level)");
    cudaStream_t s = ctx->stream;
    if (row_ptr) PSC_CUDA(cudaMemcpyAsync(row_ptr, M.ptr, sizeof(int64_t) * (M.n + 1), cudaMemcpyDeviceToHost, s));
    if (col && M.nnz) PSC_CUDA(cudaMemcpyAsync(col, M.col, sizeof(int64_t) * M.nnz, cudaMemcpyDeviceToHost, s));
    if (val && M.nnz) PSC_CUDA(cudaMemcpyAsync(val, M.val, sizeof(double) * M.nnz, cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    return PSC_OK;
  } catch (const Error& e) {
    if (ctx) ctx->err = e.what();
    return e.code;
  }
}

int psc_amg_aggregates(psc_amg* a, int level, int64_t* agg, int8_t* root) {
  psc_ctx* ctx = a ? a->ctx : nullptr;
  try {
    PSC_REQUIRE(a && level >= 0 && level < (int)a->lv.size(), PSC_ERR_ARG, "bad argument");
    const AmgLevel& L = a->lv[level];
    PSC_REQUIRE(L.agg, PSC_ERR_STATE, "no aggregation at this level (the coarsest)");
    cudaStream_t s = ctx->stream;
    if (agg) PSC_CUDA(cudaMemcpyAsync(agg, L.agg, sizeof(int64_t) * L.A.n, cudaMemcpyDeviceToHost, s));
    if (root) PSC_CUDA(cudaMemcpyAsync(root, L.root, L.A.n, cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    if (root)
      for (int64_t i = 0; i < L.A.n; ++i) root[i] = (root[i] == kRoot) ? 1 : 0;
    return PSC_OK;
  } catch (const Error& e) {
    if (ctx) ctx->err = e.what();
    return e.code;
  }
}

int psc_amg_hier_create(psc_amg* a, const psc_cycle_opts* copts, psc_hier** out) {
  psc_ctx* ctx = a ? a->ctx : nullptr;
  try {
    PSC_REQUIRE(a && out, PSC_ERR_ARG, "bad argument");
    PSC_REQUIRE(a->descs.empty(), PSC_ERR_STATE, "psc_amg_hier_create: already called for this set-up");
    const int L = (int)a->lv.size();
    cudaStream_t s = ctx->stream;
    // descriptors (one rank: no halo) and matrices straight from the device CSR
    for (int l = 0; l < L; ++l) {
      psc_desc* d = new psc_desc();
      d->ctx = ctx;
      d->n_global = a->lv[l].A.n;
      d->row_start = {0, d->n_global};
      d->own_begin = 0;
      d->n_own = d->n_global;
      a->descs.push_back(d);
    }
    auto mk = [&](const DCsr& M, psc_desc* rows, psc_desc* cols) {
      psc_mat* m = new psc_mat();
      m->ctx = ctx;
      m->rows = rows;
      m->cols = cols;
      m->n_rows = M.n;
      m->nnz = M.nnz;
      m->d_rowptr = dalloc<int64_t>(M.n + 1);
      m->d_colg = dalloc<int64_t>(M.nnz);
      m->d_valcsr = dalloc<double>(M.nnz);
      PSC_CUDA(cudaMemcpyAsync(m->d_rowptr, M.ptr, sizeof(int64_t) * (M.n + 1), cudaMemcpyDeviceToDevice, s));
      if (M.nnz) {
        PSC_CUDA(cudaMemcpyAsync(m->d_colg, M.col, sizeof(int64_t) * M.nnz, cudaMemcpyDeviceToDevice, s));
        PSC_CUDA(cudaMemcpyAsync(m->d_valcsr, M.val, sizeof(double) * M.nnz, cudaMemcpyDeviceToDevice, s));
      }
      a->mats.push_back(m);
      return m;
    };
    std::vector<psc_mat*> A(L), P(std::max(L - 1, 1)), R(std::max(L - 1, 1));
    for (int l = 0; l < L; ++l) A[l] = mk(a->lv[l].A, a->descs[l], a->descs[l]);
    // the AINV factorisation runs on the host (hier.cu ainv_factor): host copies of the
    // smoothed levels' operators, as psc_mat_create_csr keeps them (nnz <= 2^27)
    if (copts && copts->smoother == PSC_SMOOTHER_AINV)
      for (int l = 0; l + 1 < L; ++l) {
        const DCsr& M = a->lv[l].A;
        if (M.nnz > ((int64_t)1 << 27)) continue;
        psc_mat* m = A[l];
        m->h_rowptr.resize(M.n + 1);
        m->h_colg.resize(M.nnz);
        m->h_val.resize(M.nnz);
        PSC_CUDA(cudaMemcpyAsync(m->h_rowptr.data(), M.ptr, sizeof(int64_t) * (M.n + 1), cudaMemcpyDeviceToHost, s));
        if (M.nnz) {
          PSC_CUDA(cudaMemcpyAsync(m->h_colg.data(), M.col, sizeof(int64_t) * M.nnz, cudaMemcpyDeviceToHost, s));
          PSC_CUDA(cudaMemcpyAsync(m->h_val.data(), M.val, sizeof(double) * M.nnz, cudaMemcpyDeviceToHost, s));
        }
      }
    PSC_CUDA(cudaStreamSynchronize(s));
    for (int l = 0; l + 1 < L; ++l) {
      P[l] = mk(a->lv[l].P, a->descs[l], a->descs[l + 1]);
      R[l] = mk(a->lv[l].R, a->descs[l + 1], a->descs[l]);
    }
    for (psc_desc* d : a->descs) desc_assemble(d);
    for (psc_mat* m : a->mats) mat_assemble(m);
    const int rc = psc_hier_create(ctx, L, A.data(), P.data(), R.data(), copts, out);
    return rc;
  } catch (const Error& e) {
    if (ctx) ctx->err = e.what();
    return e.code;
  }
}

void psc_amg_destroy(psc_amg* a) {
  if (!a) return;
  cudaSetDevice(a->ctx->device);
  amg_free(a);
  for (psc_mat* m : a->mats) psc_mat_destroy(m);
  for (psc_desc* d : a->descs) psc_desc_destroy(d);
  delete a;
}

}  // extern "C"
