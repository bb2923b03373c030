// psc_internal.h — internal types of libpsc.so (B200 / sm_100a).
// Nothing here is part of the ABI (see include/psc.h).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "psc.h"

#include <nvtx3/nvToolsExt.h>

namespace psc {

constexpr int kSlice = 32;        // rows per sliced-ELL slice = warp size ("based on the size of a warp")
constexpr int kBlock = 256;       // threads per CTA for the row kernels (8 slices per CTA pass)
constexpr int kWarpsPerBlock = kBlock / 32;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PSC_CUDA(call)                                                                                  \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess)                                                                              \
      throw ::psc::Error(e_ == cudaErrorMemoryAllocation ? PSC_ERR_NOMEM : PSC_ERR_CUDA,                \
                         std::string(#call) + ": " + cudaGetErrorString(e_) + " @" + __FILE__ + ":" + \
                             std::to_string(__LINE__));                                                 \
  } while (0)

#define PSC_NCCL(call)                                                                                    \
  do {                                                                                                    \
    ncclResult_t r_ = (call);                                                                             \
    if (r_ != ncclSuccess)                                                                                \
      throw ::psc::Error(PSC_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_) + " @" + __FILE__ + \
                                           ":" + std::to_string(__LINE__));                               \
  } while (0)

// Device-side bounds checks of the checked build (build.py: libpsc_checked.so with
// -DPSC_CHECKS; compute-sanitizer is not available on the GPU pool): a failed check
// traps, the launch fails and the host call returns PSC_ERR_CUDA.
#ifdef PSC_CHECKS
#define PSC_DASSERT(c)     \
  do {                     \
    if (!(c)) __trap();    \
  } while (0)
#else
#define PSC_DASSERT(c) ((void)0)
#endif

#define PSC_REQUIRE(cond, code, msg)                 \
  do {                                               \
    if (!(cond)) throw ::psc::Error((code), (msg)); \
  } while (0)

template <class T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  PSC_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return static_cast<T*>(p);
}
inline void dfree(void* p) {
  if (p) cudaFree(p);
}

// Device matrix, one of two layouts chosen at assembly from the mean row length
// (DESIGN.md §5):
//  lanes == 1  sliced ELL (Hacked ELLPACK): rows grouped in 32-row
//              slices; slice s stores its width w_s = max row length of its rows
//              as a column-major w_s x 32 block of values at element offset ptr[s];
//              value k of row (32 s + lane) is at ptr[s] + 32 k + lane.  One thread
//              per row.  Column indices per slice, from cptr[s], in one of two forms:
//                ELL slice: 32 w_s explicit local columns (same layout as values);
//                DIA slice: w_s diagonal offsets shared by the 32 rows, column =
//                  local row + offset (absent entries stored as 0.0) — chosen when
//                  the slice's distinct (col - row) offsets are few (stencil-like rows,
//                  interior slices), cutting 4 B/nnz of column traffic.
//              DIA iff cptr[s+1] - cptr[s] < 32 w_s.
//  lanes == G  row groups (G in {4,8,16,32}): rows stored contiguously, each padded
//              to a multiple of G entries, ptr[i] = start of row i; G lanes of a
//              warp share one row (long rows of coarse A_l and R_l).
// Padding: value 0.0, column = the row's last valid column (0 for empty rows).
// A warp processes one "unit": a slice (lanes == 1) or 32/G consecutive rows.
struct Sell {
  int64_t n_rows = 0, n_cols_local = 0, nnz = 0, padded = 0;
  int lanes = 1;
  int64_t n_units = 0;
  int64_t* ptr = nullptr;  // lanes == 1: n_units + 1 slice offsets; else n_rows + 1 row offsets
  int64_t* cptr = nullptr; // lanes == 1: n_units + 1 column-slot offsets (ELL or DIA slices)
  int64_t col_slots = 0;   // entries of `col`
  int64_t nnz_ell = 0;     // stored nonzeros whose column index is explicit (ELL slices / row groups)
  int64_t n_dia = 0;       // DIA slices
  int64_t n_e16 = 0;       // ELL slices with 16-bit column offsets (kEll16)
  int32_t* col = nullptr;  // col_slots
  // lanes == 1: per-slice 64-byte header read by the row kernels in one coalesced
  // half-warp load (prefetched one slice ahead): [0..1] value offset, [2..3] column
  // offset, [4] width, [5] kind (0 ELL, 1 DIA), [6..13] DIA offsets, [14] DIA slot of
  // the diagonal.
  int32_t* hdr = nullptr;
  double* val = nullptr;   // padded
  // SELL-C-sigma (sorted) layouts: slot -> row and row -> slot offsets inside each
  // 256-row window (kernels.cu row_of_slot / slot_of_row); nullptr: natural order
  uint8_t* perm = nullptr;
  uint8_t* iperm = nullptr;
  int64_t* slot = nullptr;  // nnz: value slot of each CSR entry (structure-preserving updates)
  // units whose columns are all owned (interior) and the others (boundary):
  // the interior ones can run while the halo exchange is in flight.
  int32_t* interior = nullptr;
  int32_t* boundary = nullptr;
  int64_t n_interior = 0, n_boundary = 0;
  int max_width = 0;  // longest (padded) row
  int64_t max_chunk = 0;  // row groups: most entries in one chunk of 8 units (TMA ring capacity check)
  int rows_per_unit() const { return lanes == 1 ? 32 : 32 / lanes; }
};

// Per-reduction-site scratch: block partials, a ticket counter, and the slot of
// the gathered-scalar array the finalising block writes (fixed-order sums).
struct RedSite {
  double* partials = nullptr;  // [nred][grid]
  unsigned int* ticket = nullptr;
  int grid = 0;
};

}  // namespace psc

namespace psc {
// NVTX range for the host phases (visible in nsys / ncu --nvtx): set-up steps, graph
// capture, each solve
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Per-kernel device timing (psc_hier_kernel_profile): while `on`, every launcher
// brackets its launch with an event pair (recorded as graph nodes when captured)
// and files it under (name, level) with its algorithmic and layout bytes.
struct KTrace {
  struct Rec {
    const char* name;
    int level;
    double alg_bytes, layout_bytes;
    cudaEvent_t e0, e1;
  };
  bool on = false;
  int level = -1;  // hierarchy level of the launches being recorded (-1: Krylov level-0 vector ops)
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      pool.push_back(e);
    }
    return pool[used++];
  }
};
}  // namespace psc

struct psc_ctx_s {
  int rank = 0, nranks = 1, device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;       // library stream (all work)
  cudaStream_t comm_stream = nullptr;  // halo exchange stream (overlap)
  cudaStream_t user_stream = nullptr;
  cudaEvent_t ev_user = nullptr;
  ncclComm_t comm = nullptr;
  std::string err;
  int64_t launches = 0;     // kernel launch counter (incremented by every launcher)
  int64_t collectives = 0;  // NCCL call counter
  psc::KTrace kt;           // per-kernel timing (off unless profiling)
};

namespace psc {
// RAII bracket of one launch for KTrace (no-op unless ctx->kt.on)
struct KtScope {
  psc_ctx* ctx;
  cudaStream_t s;
  bool on;
  KtScope(psc_ctx* c, cudaStream_t st, const char* name, double alg, double layout) : ctx(c), s(st) {
    on = c && c->kt.on;
    if (!on) return;
    KTrace::Rec r{name, c->kt.level, alg, layout, c->kt.get(), c->kt.get()};
    PSC_CUDA(cudaEventRecordWithFlags(r.e0, s, cudaEventRecordExternal));
    c->kt.recs.push_back(r);
  }
  ~KtScope() {
    if (on) cudaEventRecordWithFlags(ctx->kt.recs.back().e1, s, cudaEventRecordExternal);
  }
};
}  // namespace psc

struct psc_desc_s {
  psc_ctx* ctx = nullptr;
  int64_t n_global = 0;
  std::vector<int64_t> row_start;
  int64_t own_begin = 0, n_own = 0;
  std::vector<int64_t> halo_req;  // registrations (unsorted, duplicates) until assembly
  bool assembled = false;
  std::vector<int64_t> halo;              // sorted unique off-rank globals
  std::vector<int64_t> rcount, roff;      // per peer: received halo entries / offset in the halo region
  std::vector<int64_t> scount, soff;      // per peer: entries sent / offset in the send list
  int64_t n_send = 0;
  int32_t* d_send_idx = nullptr;          // local owned indices to send, grouped by peer
  double* d_sendbuf = nullptr;
  int64_t* d_halo = nullptr;              // halo globals on the device (column renumbering)
  int64_t n_halo() const { return (int64_t)halo.size(); }
};

struct psc_mat_s {
  psc_ctx* ctx = nullptr;
  psc_desc* rows = nullptr;
  psc_desc* cols = nullptr;
  int64_t n_rows = 0, nnz = 0;
  // staged device CSR (global columns) until assembly
  int64_t* d_rowptr = nullptr;
  int64_t* d_colg = nullptr;
  double* d_valcsr = nullptr;
  bool assembled = false;
  psc::Sell S;
  // host copy of this rank's rows (global columns), kept for small matrices only:
  // used to replicate the coarsest level on every rank.
  std::vector<int64_t> h_rowptr, h_colg;
  std::vector<double> h_val;
};

namespace psc {
// ctx_desc.cu
void halo_exchange(psc_ctx* ctx, psc_desc* d, double* x, cudaStream_t s);
void desc_assemble(psc_desc* d);
// mat.cu
void mat_assemble(psc_mat* m);
}  // namespace psc
