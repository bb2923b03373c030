// hier.cu — AMG hierarchy handle, V-cycle (Eq. (2)) and PCG driver of libpsc.so.
//
// One PCG iteration = one CUDA Graph launch (V-cycle + p update + q = A p +
// x/r update + the 2-scalar device->host copy); the host waits once per
// iteration for the stopping test (P:314 relative residual), so the only
// per-iteration host<->device traffic is 2*nranks doubles.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include "kernels.h"
#include "p2p.h"

using namespace psc;

namespace {

// vectors of the solve path: padded so TMA bulk copies of the last rows may overread
double* dvec(int64_t n) { return dalloc<double>((size_t)n + 64); }

// Gathered per-rank partial scalars (slot-major, nranks entries each).  Main
// Krylov loop: (p, Ap), (r, r), (r, z) [FCG: (z, A p_old)], (b, b), FCG (p, r).
// Coarsest PCG (general form): (p, Ap), (r, r), (r, z) double-buffered by
// iteration parity, (b, b).  Every slot is read before a peer can write its
// next value: between a read and the peer's next push lies an all-gather that
// needs this rank's later contribution.
enum Slot {
  S_PQ = 0, S_RR = 1, S_RZ = 2, S_BB = 3, S_PR = 4,
  S_CPQ = 5, S_CRR = 6, S_CZ0 = 7, S_CZ1 = 8, S_CBB = 9,
  NSLOT = 10
};

struct LevelWS {
  psc_mat *A = nullptr, *P = nullptr, *R = nullptr;
  psc_desc* d = nullptr;      // nullptr: replicated level (no halo, no exchange)
  int64_t n = 0, nh = 0;
  double* dinv = nullptr;     // n
  double* x[2] = {nullptr, nullptr};  // n + nh
  double* r = nullptr;        // n + nh
  double* b = nullptr;        // n (level >= 1: R_{l-1} r_{l-1})
  // coarsest-level solver data (last level of a level array)
  double* dense = nullptr;    // n x n row-major copy of A when n <= coarse_dense_max_rows()
  bool one_cta = false;       // sparse one-CTA solver applies
  double* cz = nullptr;       // general coarsest PCG: z and q = A p (n)
  double* cq = nullptr;
  // AINV smoother: M^-1 = Z D^-1 Z^T; Z and Z^T as sliced ELL, 1/p, scratch
  bool ainv = false;
  Sell Z, Zt;
  double* ainv_dinv = nullptr;
  double* az_t = nullptr;
  double* az_u = nullptr;
};

// Replicated suffix (nranks > 1): levels first..L-1 are held whole on every
// rank.  The V-cycle gathers b at level `first` once (all-gather), runs the
// rest of the cycle redundantly with no halo exchange (row results are the same
// arithmetic as the distributed sweeps), and scatters x to the owned+halo slots
// of level `first`.  The coarse levels are latency-bound (one exchange costs
// ~10 us, about a whole coarse kernel), so this removes ~2 x 10 exchanges per
// V-cycle at the price of kernels over a few thousand more rows.
struct Replica {
  bool on = false;
  int first = -1;
  int64_t N = 0, maxcnt = 0;    // global rows of level `first`; all-gather block per rank
  std::vector<LevelWS> lv;      // replicated levels first..L-1 (global numbering, internal matrices)
  std::vector<psc_mat*> mats;   // owned internal matrices
  double* sendbuf = nullptr;    // maxcnt
  double* gbuf = nullptr;       // nranks * maxcnt (in the arena: peers write it)
  int64_t* map_full = nullptr;  // N: global g -> position in gbuf
  int64_t* map_loc = nullptr;   // n + nh of level `first`: local slot -> global index
};

}  // namespace

struct psc_hier_s {
  psc_ctx* ctx = nullptr;
  int L = 0;
  psc_cycle_opts opt{4, 4, 30, PSC_COARSE_SWEEPS, 40, 1e-10, 0};
  std::vector<LevelWS> lv;
  Replica rep;
  // dense suffix: the V-cycle operator of levels dsuf_l.. of the level array
  // *dsuf_lv, precomputed as a dense row-major matrix (linear coarse solver only)
  const std::vector<LevelWS>* dsuf_lv = nullptr;
  int dsuf_l = -1;
  double* dsuf = nullptr;
  // CG state (level 0)
  double* x_int = nullptr;  // n0 + nh0
  double* r_cg = nullptr;   // n0
  double* p = nullptr;      // n0 + nh0
  double* q = nullptr;      // n0
  double* d_scal = nullptr; // NSLOT * nranks gathered partial scalars, then rz_old
  double* h_scal = nullptr; // pinned mirror
  double* d_bhost = nullptr;  // device staging for psc_pcg_solve_host
  double* d_xhost = nullptr;
  RedSite red1, red2;
  int* d_done = nullptr;        // stop flag of the general coarsest PCG
  // weight of the (., z) reduction in the last level-0 post-sweep while an FCG
  // iteration is recorded (q = A p_old); nullptr: r (PCG)
  const double* rz_weight = nullptr;
  // fused push: the vector whose halo the last row kernel pushed, and the launch count
  // right after it (the push is consumed only by the immediately next launch)
  const double* pushed = nullptr;
  int64_t pushed_at = -1;
  // graph of one Krylov iteration, per method (PSC_KRYLOV_PCG, PSC_KRYLOV_FCG)
  cudaGraphExec_t iter_exec[2] = {nullptr, nullptr};
  cudaGraphExec_t prof_exec[2] = {nullptr, nullptr};  // the same iteration with per-kernel event pairs
  int64_t iter_launches[2] = {0, 0}, iter_collectives[2] = {0, 0};
  double* z_ptr = nullptr;
  // dominant-kernel timing (level-0 l1-Jacobi sweep) inside the graph
  std::vector<cudaEvent_t> ev_dom;  // pairs (start, end)
  int dom_used = 0;
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // exchange / interior overlap (run_rows)
  // buffers peers write into (halo-bearing vectors, gathered scalars, coarse
  // gather buffer, P2P flags) live in one arena: one CUDA IPC handle maps them
  char* arena = nullptr;
  P2P p2p;
};

namespace {

thread_local std::string g_herr;

int hfail(psc_ctx* ctx, const Error& e) {
  if (ctx) ctx->err = e.what();
  g_herr = e.what();
  return e.code;
}

void enter(psc_ctx* ctx) {
  PSC_CUDA(cudaSetDevice(ctx->device));
  PSC_CUDA(cudaEventRecord(ctx->ev_user, ctx->user_stream));
  PSC_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_user, 0));
}

double* scal(psc_hier* h, Slot s) { return h->d_scal + (size_t)s * h->ctx->nranks; }
double* scal_mine(psc_hier* h, Slot s) { return scal(h, s) + h->ctx->rank; }
double* rz_old(psc_hier* h) { return h->d_scal + (size_t)NSLOT * h->ctx->nranks; }

void allgather_slot(psc_hier* h, Slot s, cudaStream_t st) {
  psc_ctx* ctx = h->ctx;
  if (ctx->nranks == 1) return;
  if (p2p_allgather(ctx, h->p2p, scal_mine(h, s), 1, scal(h, s), st)) return;
  PSC_NCCL(ncclAllGather(scal_mine(h, s), scal(h, s), 1, ncclDouble, ctx->comm, st));
  ctx->collectives++;
}

// halo exchange of a level vector: NVLink peer stores when available, else NCCL
void exchange(psc_hier* h, psc_desc* d, double* x, cudaStream_t s) {
  psc_ctx* ctx = h->ctx;
  if (ctx->nranks == 1) return;

  if (p2p_halo(ctx, h->p2p, d, x, s)) return;
  halo_exchange(ctx, d, x, s);
}

// Halo exchange of a.x before the row kernel `a` is launched.
void prep(psc_hier* h, psc_desc* d, RowArgs& a, cudaStream_t s) {
  psc_ctx* ctx = h->ctx;
  if (ctx->nranks == 1 || !d) return;
  // TIMING EXPERIMENTS ONLY (wrong results): PSC_DEBUG_SKIP_HALO=1 skips halo exchanges
  static const bool skip = getenv("PSC_DEBUG_SKIP_HALO") != nullptr;
  static const int skip_from = getenv("PSC_DEBUG_SKIP_HALO_FROM") ? atoi(getenv("PSC_DEBUG_SKIP_HALO_FROM")) : 1 << 30;
  if (skip) return;
  for (int l = skip_from; l < h->L; ++l)
    if (h->lv[l].d == d) return;
  // TIMING EXPERIMENTS ONLY: PSC_DEBUG_DOUBLE_HALO=1 adds a second, standalone exchange
  static const bool twice = getenv("PSC_DEBUG_DOUBLE_HALO") != nullptr;
  if (twice) exchange(h, d, const_cast<double*>(a.x), s);
  exchange(h, d, const_cast<double*>(a.x), s);
}

// A row kernel whose input x needs a halo exchange first.  Distributed levels
// (non-reducing kernels): the exchange runs on the communication stream while the
// interior chunks (no halo column) run on the main stream; the boundary chunks
// follow once the exchange has landed — the exchange (~10 us) hides behind the
// interior work instead of preceding it.  Otherwise: prep() + one launch.
// Opt-in (PSC_OVERLAP=1): measured slower on 2 B200 (6122 vs 6555 Mdof*iters/s at
// 256^3/GPU): the split adds a launch and a join per kernel (92 -> 120 launches per
// iteration), which costs more than the ~10 us exchange it hides.
// Fused push (opt-in PSC_PUSH=1): a producer row kernel pushes its
// output's boundary rows into the neighbours' halo slots and signals; the next launch,
// when it is the row kernel reading that vector's halo, waits instead of a stand-alone
// exchange.  Measured slower on 2 B200 (6670 vs 7050 Mdof*iters/s): producer-end
// system fences and consumer-start waits serialise the kernels on NVLink latency.  push_d: the output's row space when the caller's next launch reads the
// output's halo (nullptr: no push).
bool fused_push_on() {
  static const bool on = getenv("PSC_PUSH") != nullptr && getenv("PSC_OVERLAP") == nullptr &&
                         getenv("PSC_DEBUG_SKIP_HALO") == nullptr && getenv("PSC_DEBUG_DOUBLE_HALO") == nullptr &&
                         getenv("PSC_DEBUG_POISON_HALO") == nullptr;
  return on;
}

// TEST HOOK ("halo freshness"): PSC_DEBUG_POISON_HALO=1 fills the halo slots
// of x with NaN (all-ones bytes) right after every kernel that read them; a later kernel
// reading them without a new exchange would carry the NaN into the owned results.
// (After the read, not before the exchange: a peer may push into the halo before this
// rank's own exchange kernel starts.)
void poison_halo(psc_hier* h, psc_desc* d, const double* x, cudaStream_t s) {
  static const bool poison = getenv("PSC_DEBUG_POISON_HALO") != nullptr;
  if (poison && h->ctx->nranks > 1 && d && d->n_halo() > 0)
    PSC_CUDA(cudaMemsetAsync(const_cast<double*>(x) + d->n_own, 0xFF, sizeof(double) * d->n_halo(), s));
}

// tev: optional event pair recorded around the row kernel alone (after its halo
// exchange: the dominant-kernel timing must not include the wait for the neighbours)
void run_rows(psc_hier* h, psc_desc* d, const Sell& S, RowOp op, RowArgs& a, cudaStream_t s,
              psc_desc* push_d = nullptr, cudaEvent_t* tev = nullptr) {
  psc_ctx* ctx = h->ctx;
  // a pushed halo is only valid for the immediately following launch
  const bool pushed_here = h->pushed && h->pushed == a.x && h->pushed_at == ctx->launches + ctx->collectives;
  h->pushed = nullptr;
  static const bool no_overlap = getenv("PSC_OVERLAP") == nullptr || getenv("PSC_DEBUG_SKIP_HALO") != nullptr ||
                                 getenv("PSC_DEBUG_SKIP_HALO_FROM") != nullptr ||
                                 getenv("PSC_DEBUG_DOUBLE_HALO") != nullptr;
  const bool reduces = (op == RowOp::SpmvDot || op == RowOp::SweepDot || op == RowOp::ResidDot2);
  if (!no_overlap && ctx->nranks > 1 && d && !reduces && S.n_boundary > 0 && S.n_interior > 0) {
    PSC_CUDA(cudaEventRecord(h->ev_fork, s));
    PSC_CUDA(cudaStreamWaitEvent(ctx->comm_stream, h->ev_fork, 0));
    exchange(h, d, const_cast<double*>(a.x), ctx->comm_stream);
    PSC_CUDA(cudaEventRecord(h->ev_join, ctx->comm_stream));
    if (tev) PSC_CUDA(cudaEventRecordWithFlags(tev[0], s, cudaEventRecordExternal));
    launch_rows(ctx, S, op, a, s, SliceSet::Interior);
    PSC_CUDA(cudaStreamWaitEvent(s, h->ev_join, 0));
    launch_rows(ctx, S, op, a, s, SliceSet::Boundary);
    if (tev) PSC_CUDA(cudaEventRecordWithFlags(tev[1], s, cudaEventRecordExternal));
    poison_halo(h, d, a.x, s);
    return;
  }
  if (!(pushed_here && d && rows_can_push(S, a) && p2p_wait_spec(ctx, h->p2p, a.x, a.wait))) prep(h, d, a, s);
  const bool push = fused_push_on() && push_d && ctx->nranks > 1 && rows_can_push(S, a) &&
                    p2p_push_spec(ctx, h->p2p, push_d, a.y, a.push);
  if (tev) PSC_CUDA(cudaEventRecordWithFlags(tev[0], s, cudaEventRecordExternal));
  launch_rows(ctx, S, op, a, s);
  if (tev) PSC_CUDA(cudaEventRecordWithFlags(tev[1], s, cudaEventRecordExternal));
  if (push) {
    h->pushed = a.y;
    h->pushed_at = ctx->launches + ctx->collectives;
  }
  poison_halo(h, d, a.x, s);
}

// ------------------------------------------------------------ coarsest level
// `nsweeps` l1-Jacobi sweeps from zero on the last level of a level
// array.  Returns its iterate.
double* coarse_sweeps(psc_hier* h, LevelWS& W, const double* b, int nsweeps, cudaStream_t s) {
  psc_ctx* ctx = h->ctx;
  if (W.dense) {
    launch_coarse_dense(ctx, W.dense, W.n, W.dinv, b, W.x[0], nsweeps, s);
    return W.x[0];
  }
  if (W.one_cta) {
    launch_coarse_solve(ctx, W.A->S, W.dinv, b, W.x[0], nsweeps, s);
    return W.x[0];
  }
  // general path: sweeps, one halo exchange each when distributed
  int cur = 0;
  if (nsweeps <= 0) {
    PSC_CUDA(cudaMemsetAsync(W.x[0], 0, sizeof(double) * (W.n + W.nh), s));
    return W.x[0];
  }
  launch_scale(ctx, W.n, W.dinv, b, W.x[0], s);
  for (int k = 1; k < nsweeps; ++k) {
    RowArgs a;
    a.vec_padded = true;  // library buffers, padded (dvec)
    a.x = W.x[cur];
    a.b = b;
    a.dinv = W.dinv;
    a.y = W.x[cur ^ 1];
    run_rows(h, W.d, W.A->S, RowOp::Sweep, a, s);
    cur ^= 1;
  }
  return W.x[cur];
}

// PCG from zero with the l1-Jacobi preconditioner, at most coarse_maxit
// iterations, stopping at ||r|| <= coarse_tol ||b|| (reading R23).
// Dense one-CTA kernel when the level has a dense copy; otherwise one SpMV +
// two vector kernels per iteration, all recorded (the device flag h->d_done
// makes the steps after convergence no-ops), with all-gathers of the partial
// scalars when the level is distributed.  x in W.x[0], p in W.x[1] (halo-
// bearing: exchanged before each SpMV), r in W.r.
double* coarse_pcg(psc_hier* h, LevelWS& W, const double* b, cudaStream_t s) {
  psc_ctx* ctx = h->ctx;
  const int maxit = h->opt.coarse_maxit;
  const double tol = h->opt.coarse_tol;
  if (W.dense) {
    launch_coarse_dense_pcg(ctx, W.dense, W.n, W.dinv, b, W.x[0], maxit, tol, s);
    return W.x[0];
  }
  const int R = ctx->nranks;
  const bool dist = W.d && R > 1;
  const int nr = dist ? R : 1;
  auto g = [&](Slot sl) { return dist ? scal(h, sl) : scal_mine(h, sl); };
  double *x = W.x[0], *p = W.x[1], *r = W.r, *z = W.cz, *q = W.cq;
  launch_cpcg_init(ctx, W.n, b, W.dinv, x, r, z, p, h->d_done, &h->red2, scal_mine(h, S_CZ0), (S_CBB - S_CZ0) * R,
                   s);
  if (dist) {
    allgather_slot(h, S_CZ0, s);
    allgather_slot(h, S_CBB, s);
  }
  for (int k = 1; k <= maxit; ++k) {
    const Slot zo = (k & 1) ? S_CZ0 : S_CZ1;  // (r, z) of iteration k-1
    const Slot zn = (k & 1) ? S_CZ1 : S_CZ0;  // (r, z) of iteration k
    {
      RowArgs a;
      a.vec_padded = true;
      a.x = p;
      a.y = q;
      a.red = &h->red1;
      a.red_out = scal_mine(h, S_CPQ);
      prep(h, W.d, a, s);
      launch_rows(ctx, W.A->S, RowOp::SpmvDot, a, s);
      poison_halo(h, W.d, a.x, s);
    }
    if (dist) allgather_slot(h, S_CPQ, s);
    launch_cpcg_update(ctx, W.n, x, p, r, q, z, W.dinv, g(S_CPQ), g(zo), nr, h->d_done, &h->red2,
                       scal_mine(h, S_CRR), (zn - S_CRR) * R, s);
    if (dist) {
      allgather_slot(h, S_CRR, s);
      allgather_slot(h, zn, s);
    }
    if (k < maxit) launch_cpcg_dir(ctx, W.n, z, p, g(S_CRR), g(S_CBB), g(zn), g(zo), nr, tol, h->d_done, s);
  }
  return x;
}

// B_ell: the configured coarsest-level solver
double* coarse_solve(psc_hier* h, LevelWS& W, const double* b, cudaStream_t s) {
  if (h->opt.coarse_solver == PSC_COARSE_PCG) return coarse_pcg(h, W, b, s);
  return coarse_sweeps(h, W, b, h->opt.coarse_sweeps, s);
}

// nsweeps l1-Jacobi sweeps from zero on W (pre-smoothing: the rightmost factor
// of Eq. (2) applied `pre` times).  The first sweep is x = M^{-1} b exactly;
// first_done: x[0] = M^{-1} b was already written by the kernel that produced b
// (the restriction, or the CG update at level 0).  Returns the buffer index of x.
// timing: event pairs around level-0 sweeps (dominant kernel, measured live).
void free_ainv(LevelWS& W) {
  sell_free(W.Z);
  sell_free(W.Zt);
  dfree(W.ainv_dinv);
  dfree(W.az_t);
  dfree(W.az_u);
  W.ainv_dinv = W.az_t = W.az_u = nullptr;
  W.ainv = false;
}

// ------------------------------------------------------------ AINV smoother
// Incomplete A-biconjugation (reading R27): A symmetric positive definite,
// W = Z, A^-1 ~ Z D^-1 Z^T.  Right-looking: z_j = e_j; for i = 0..n-1: p_i = a_i^T z_i,
// and for every j > i with p_j = a_i^T z_j != 0: z_j -= (p_j / p_i) z_i, dropping the
// updated entries below drop_tol (never z_jj).  Only columns j whose z_j has an entry
// in the pattern of row i can have p_j != 0, so the candidates come from a row ->
// columns index of Z.  Sums run over row i's entries in column order; one rounding
// per operation (host code built with -ffp-contract=off).  Host work at set-up.
void ainv_factor(int64_t n, const int64_t* ptr, const int64_t* col, const double* val, double drop,
                 std::vector<int64_t>& zptr, std::vector<int64_t>& zrow, std::vector<double>& zval,
                 std::vector<double>& p) {
  std::vector<std::vector<std::pair<int64_t, double>>> z(n);  // column j: (row k, z_kj), rows increasing
  std::vector<std::vector<int64_t>> cols_at(n);                // row k -> columns j with z_kj present (or once)
  for (int64_t j = 0; j < n; ++j) {
    z[j].push_back({j, 1.0});
    cols_at[j].push_back(j);
  }
  p.assign(n, 0.0);
  auto dot_row = [&](int64_t i, const std::vector<std::pair<int64_t, double>>& zj) {
    double s = 0.0;
    size_t q = 0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {  // row i in column order
      const int64_t c = col[k];
      while (q < zj.size() && zj[q].first < c) ++q;
      if (q < zj.size() && zj[q].first == c) s = s + val[k] * zj[q].second;
    }
    return s;
  };
  std::vector<int64_t> cand;
  std::vector<std::pair<int64_t, double>> merged;
  for (int64_t i = 0; i < n; ++i) {
    const double pi = dot_row(i, z[i]);
    PSC_REQUIRE(pi > 0.0, PSC_ERR_STATE, "AINV breakdown: pivot " + std::to_string(i) + " <= 0");
    p[i] = pi;
    cand.clear();
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k)
      for (int64_t j : cols_at[col[k]])
        if (j > i) cand.push_back(j);
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    const auto& zi = z[i];
    for (int64_t j : cand) {
      const double pj = dot_row(i, z[j]);
      if (pj == 0.0) continue;
      const double f = pj / pi;
      // z_j - f z_i over the rows of z_i (z_i has rows <= i < j, so z_jj stays 1)
      merged.clear();
      const auto& zj = z[j];
      size_t a = 0, b = 0;
      while (a < zj.size() || b < zi.size()) {
        if (b == zi.size() || (a < zj.size() && zj[a].first < zi[b].first)) {
          merged.push_back(zj[a++]);
        } else {
          const int64_t k = zi[b].first;
          const bool have = a < zj.size() && zj[a].first == k;
          const double v = (have ? zj[a].second : 0.0) - f * zi[b].second;
          if (have) ++a;
          ++b;
          if (k == j || std::fabs(v) >= drop) {
            merged.push_back({k, v});
            if (!have) cols_at[k].push_back(j);
          }
        }
      }
      z[j].swap(merged);
    }
  }
  zptr.assign(n + 1, 0);  // Z by rows: (k, j)
  for (int64_t j = 0; j < n; ++j)
    for (auto& e : z[j]) zptr[e.first + 1]++;
  for (int64_t k = 0; k < n; ++k) zptr[k + 1] += zptr[k];
  zrow.assign(zptr[n], 0);
  zval.assign(zptr[n], 0.0);
  std::vector<int64_t> fill(zptr.begin(), zptr.end() - 1);
  for (int64_t j = 0; j < n; ++j)  // columns in increasing j: each row of Z comes out sorted
    for (auto& e : z[j]) {
      const int64_t o = fill[e.first]++;
      zrow[o] = j;
      zval[o] = e.second;
    }
}

// device copy of a host CSR (local columns) as sliced ELL
void sell_from_host(psc_ctx* ctx, int64_t n, int64_t ncols, const std::vector<int64_t>& ptr,
                    const std::vector<int64_t>& col, const std::vector<double>& val, Sell& S) {
  cudaStream_t s = ctx->stream;
  const int64_t nnz = ptr[n];
  // rows in column order, so that the layout can use DIA slices (AINV factors of a
  // stencil matrix are a few diagonals: Z of 7-point Poisson at drop 0.1 has offsets
  // 0, 1, nx, nx*ny) -- the SpMV's per-row summation order is then the column order
  std::vector<int64_t> sc(col);
  std::vector<double> sv(val);
  std::vector<std::pair<int64_t, double>> tmp;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t b = ptr[i], e = ptr[i + 1];
    if (std::is_sorted(sc.begin() + b, sc.begin() + e)) continue;
    tmp.clear();
    for (int64_t k = b; k < e; ++k) tmp.emplace_back(sc[k], sv[k]);
    std::stable_sort(tmp.begin(), tmp.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    for (int64_t k = b; k < e; ++k) {
      sc[k] = tmp[k - b].first;
      sv[k] = tmp[k - b].second;
    }
  }
  int64_t* dp = dalloc<int64_t>(n + 1);
  int64_t* dc = dalloc<int64_t>(nnz);
  double* dv = dalloc<double>(nnz);
  PSC_CUDA(cudaMemcpyAsync(dp, ptr.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  if (nnz) {
    PSC_CUDA(cudaMemcpyAsync(dc, sc.data(), sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, s));
    PSC_CUDA(cudaMemcpyAsync(dv, sv.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
  }
  sell_from_csr(ctx, n, dp, dc, dv, nnz, 0, ncols, nullptr, 0, S, s, 0, true);
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(dp);
  dfree(dc);
  dfree(dv);
}

// AINV factors of level W from its matrix's host copy.  Distributed level: the owned
// diagonal block (columns outside this rank's rows dropped: the paper's block-Jacobi
// form); replicated level or one rank: the whole matrix.
void build_ainv(psc_hier* h, LevelWS& W) {
  psc_mat* A = W.A;
  PSC_REQUIRE((int64_t)A->h_rowptr.size() == A->n_rows + 1, PSC_ERR_STATE,
              "AINV smoother needs the matrix's host copy (nnz <= 2^27)");
  free_ainv(W);
  const int64_t n = W.n;
  const int64_t ob = W.d ? W.d->own_begin : 0;
  std::vector<int64_t> bp(n + 1, 0), bc;
  std::vector<double> bv;
  for (int64_t i = 0; i < n; ++i) {  // the block in local numbering, columns in order
    for (int64_t k = A->h_rowptr[i]; k < A->h_rowptr[i + 1]; ++k) {
      const int64_t c = A->h_colg[k] - ob;
      if (c < 0 || c >= n) continue;
      bc.push_back(c);
      bv.push_back(A->h_val[k]);
    }
    bp[i + 1] = (int64_t)bc.size();
  }
  std::vector<int64_t> zp, zr, tp, tr;
  std::vector<double> zv, tv, pv;
  ainv_factor(n, bp.data(), bc.data(), bv.data(), h->opt.ainv_drop, zp, zr, zv, pv);
  // Z^T by rows (= columns of Z)
  tp.assign(n + 1, 0);
  for (int64_t q = 0; q < zp[n]; ++q) tp[zr[q] + 1]++;
  for (int64_t j = 0; j < n; ++j) tp[j + 1] += tp[j];
  tr.assign(zp[n], 0);
  tv.assign(zp[n], 0.0);
  std::vector<int64_t> fill(tp.begin(), tp.end() - 1);
  for (int64_t k = 0; k < n; ++k)
    for (int64_t q = zp[k]; q < zp[k + 1]; ++q) {
      const int64_t o = fill[zr[q]]++;
      tr[o] = k;
      tv[o] = zv[q];
    }
  sell_from_host(h->ctx, n, n, zp, zr, zv, W.Z);
  sell_from_host(h->ctx, n, n, tp, tr, tv, W.Zt);
  std::vector<double> dinv(n);
  for (int64_t i = 0; i < n; ++i) dinv[i] = 1.0 / pv[i];
  W.ainv_dinv = dvec(n);
  W.az_t = dvec(n);
  W.az_u = dvec(n);
  PSC_CUDA(cudaMemcpy(W.ainv_dinv, dinv.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
  W.ainv = true;
}

// One AINV sweep in place: x += Z D^-1 Z^T (b - A x); from_zero: x = Z D^-1 Z^T b
void ainv_sweep(psc_hier* h, LevelWS& W, const double* b, double* x, bool from_zero, cudaStream_t s) {
  psc_ctx* ctx = h->ctx;
  const double* r = b;
  if (!from_zero) {
    RowArgs a;
    a.vec_padded = true;
    a.x = x;
    a.b = b;
    a.y = W.r;
    run_rows(h, W.d, W.A->S, RowOp::Resid, a, s);
    r = W.r;
  }
  {  // u = D^-1 Z^T r  (the Spmv epilogue's second output y2 = dinv2 .* y)
    RowArgs a;
    a.vec_padded = true;
    a.x = r;
    a.y = W.az_t;
    a.y2 = W.az_u;
    a.dinv2 = W.ainv_dinv;
    launch_rows(ctx, W.Zt, RowOp::Spmv, a, s);
  }
  RowArgs a;
  a.vec_padded = true;
  a.x = W.az_u;
  a.y = x;
  launch_rows(ctx, W.Z, from_zero ? RowOp::Spmv : RowOp::PAdd, a, s);
}

// PSC_NO_FUSED_SCALE=1: every first sweep from zero is a stand-alone x = M^-1 b launch
bool fuse_first_sweep() { return getenv("PSC_NO_FUSED_SCALE") == nullptr; }

int pre_smooth(psc_hier* h, LevelWS& W, const double* b, int nsweeps, cudaStream_t s, bool timing,
               bool first_done = false) {
  psc_ctx* ctx = h->ctx;
  if (nsweeps <= 0) {
    PSC_CUDA(cudaMemsetAsync(W.x[0], 0, sizeof(double) * (W.n + W.nh), s));
    return 0;
  }
  if (W.ainv) {  // AINV sweeps in place in x[0] (first_done never set for AINV levels)
    for (int k = 0; k < nsweeps; ++k) ainv_sweep(h, W, b, W.x[0], k == 0, s);
    return 0;
  }
  int cur = 0, k = 1;
  if (!first_done) {
    if (nsweeps >= 2 && W.nh == 0 && (h->ctx->nranks == 1 || !W.d) && fuse_first_sweep()) {
      // the first two sweeps from zero in one pass (RowOp::Sweep0): x1 = M^-1 b is
      // formed where it is gathered, never stored (no halo: single rank or replicated)
      RowArgs a;
      a.vec_padded = true;
      a.x = W.x[0];  // scratch of the two-launch fallback
      a.b = b;
      a.dinv = W.dinv;
      a.y = W.x[1];
      launch_rows(ctx, W.A->S, RowOp::Sweep0, a, s);
      cur = 1;
      k = 2;
    } else {
      launch_scale(ctx, W.n, W.dinv, b, W.x[0], s);
    }
  }
  for (; k < nsweeps; ++k) {
    RowArgs a;
    a.vec_padded = true;  // library buffers, padded (dvec)
    a.x = W.x[cur];
    a.b = b;
    a.dinv = W.dinv;
    a.y = W.x[cur ^ 1];
    const bool t = timing && h->dom_used + 2 <= (int)h->ev_dom.size();
    // output read next by the following sweep or by the residual (both row kernels)
    run_rows(h, W.d, W.A->S, RowOp::Sweep, a, s, W.d, t ? &h->ev_dom[h->dom_used] : nullptr);
    if (t) h->dom_used += 2;
    cur ^= 1;
  }
  return cur;
}


// Smoothing sweeps at hierarchy level `glev`: the base count, doubled per level
// for the variable V-cycle (P:330 footnote, reading R25).
int level_sweeps(const psc_hier* h, int base, int glev) { return h->opt.variable_v ? base << glev : base; }

double* vcycle_rec(psc_hier* h, std::vector<LevelWS>& LV, int l, const double* b, cudaStream_t s, bool timing,
                   bool first_done, bool dist);

// The replicated suffix: gather b of level `first`, cycle on the whole coarse
// hierarchy, scatter x to the owned+halo slots of level `first`.
double* replicated_cycle(psc_hier* h, const double* b, cudaStream_t s) {
  psc_ctx* ctx = h->ctx;
  Replica& R = h->rep;
  LevelWS& W = h->lv[R.first];
  if (!p2p_allgather(ctx, h->p2p, b, W.n, R.gbuf, s)) {
    if (W.n) PSC_CUDA(cudaMemcpyAsync(R.sendbuf, b, sizeof(double) * W.n, cudaMemcpyDeviceToDevice, s));
    PSC_NCCL(ncclAllGather(R.sendbuf, R.gbuf, R.maxcnt, ncclDouble, ctx->comm, s));
    ctx->collectives++;
  }
  launch_gather(ctx, R.N, R.map_full, R.gbuf, R.lv[0].b, s);
  double* xf = vcycle_rec(h, R.lv, 0, R.lv[0].b, s, false, false, false);
  launch_gather(ctx, W.n + W.nh, R.map_loc, xf, W.x[0], s);
  return W.x[0];
}

// z = B_l b  (Eq. (2)), recursively over the level array LV (the
// distributed levels, or the replicated suffix when dist == false).  At level
// 0 the last post-sweep also accumulates (b, z) = (r, z) into slot S_RZ.
double* vcycle_rec(psc_hier* h, std::vector<LevelWS>& LV, int l, const double* b, cudaStream_t s, bool timing,
                   bool first_done, bool dist) {
  psc_ctx* ctx = h->ctx;
  const int Lend = (int)LV.size();
  // hierarchy level of LV[l] (the replicated suffix starts at level rep.first)
  const int glev = l + (&LV == &h->rep.lv ? h->rep.first : 0);
  ctx->kt.level = glev;
  if (dist && h->rep.on && l == h->rep.first) return replicated_cycle(h, b, s);
  if (h->dsuf && &LV == h->dsuf_lv && l == h->dsuf_l) {  // the whole sub-cycle as one dense product
    launch_dense_gemv(ctx, h->dsuf, LV[l].n, b, LV[l].x[0], s);
    return LV[l].x[0];
  }
  if (l == Lend - 1) {
    double* xc = coarse_solve(h, LV[l], b, s);
    // a one-level hierarchy: the coarsest solver is the whole V-cycle, so (r, z) of
    // the Krylov iteration is reduced here (otherwise by the last level-0 post-sweep)
    if (dist && l == 0)
      launch_dot(ctx, LV[0].n, h->rz_weight ? h->rz_weight : b, xc, &h->red1, scal_mine(h, S_RZ), s);
    return xc;
  }
  LevelWS& W = LV[l];
  LevelWS& C = LV[l + 1];
  const bool time_here = timing && dist && l == 0;
  const bool next_replicated = dist && h->rep.on && l + 1 == h->rep.first;
  // (I - M^-1 A)^pre, then the coarse-grid correction (I - P B_{l+1} P^T A):
  // r = b - A x ; b_c = R r ; x += P B_{l+1} b_c
  const int pre = level_sweeps(h, h->opt.pre_sweeps, glev);
  int cur = pre_smooth(h, W, b, pre, s, time_here, first_done);
  {
    RowArgs a;
    a.vec_padded = true;  // library buffers, padded (dvec)
    a.x = W.x[cur];
    a.b = b;
    a.y = W.r;
    RowArgs ra;  // the restriction, which reads r's halo next
    ra.vec_padded = true;
    run_rows(h, W.d, W.A->S, RowOp::Resid, a, s, rows_can_push(W.R->S, ra) ? W.d : nullptr);
  }
  // fused: the next level's first sweep from zero, x_{l+1} = M^{-1} b_{l+1}
  const bool next_dense = h->dsuf && &LV == h->dsuf_lv && l + 1 == h->dsuf_l;
  const bool fuse = fuse_first_sweep() && l + 1 < Lend - 1 && h->opt.pre_sweeps > 0 && !next_replicated &&
                    !next_dense && !C.ainv;
  {
    RowArgs a;
    a.vec_padded = true;  // library buffers, padded (dvec)
    a.x = W.r;
    a.y = C.b;
    if (fuse) {
      a.y2 = C.x[0];
      a.dinv2 = C.dinv;
    }
    run_rows(h, W.d, W.R->S, RowOp::Spmv, a, s);
  }
  double* xc = vcycle_rec(h, LV, l + 1, C.b, s, timing, fuse, dist);
  ctx->kt.level = glev;
  {
    RowArgs a;
    a.vec_padded = true;  // library buffers, padded (dvec)
    a.x = xc;
    a.y = W.x[cur];
    if (next_replicated) launch_rows(ctx, W.P->S, RowOp::PAdd, a, s);  // the replicated cycle filled xc's halo
    else run_rows(h, C.d, W.P->S, RowOp::PAdd, a, s, W.d);  // x's halo read next by the first post-sweep
  }
  // (I - M^-T A)^post ; M diagonal so M^-T = M^-1
  const int post = level_sweeps(h, h->opt.post_sweeps, glev);
  const bool level0 = dist && l == 0;
  if (W.ainv) {
    for (int k = 0; k < post; ++k) ainv_sweep(h, W, b, W.x[cur], false, s);
    if (level0)
      launch_dot(ctx, W.n, h->rz_weight ? h->rz_weight : b, W.x[cur], &h->red1, scal_mine(h, S_RZ), s);
    return W.x[cur];
  }
  for (int k = 0; k < post; ++k) {
    const bool last0 = (level0 && k == post - 1);
    RowArgs a;
    a.vec_padded = true;  // library buffers, padded (dvec)
    a.x = W.x[cur];
    a.b = b;
    a.dinv = W.dinv;
    a.y = W.x[cur ^ 1];
    if (last0) {
      a.red = &h->red1;
      a.red_out = scal_mine(h, S_RZ);
      a.w = h->rz_weight;
    }
    const bool t = time_here && h->dom_used + 2 <= (int)h->ev_dom.size();
    // the output's halo is read next by the following post-sweep, or (last sweep,
    // level >= 1) by the prolongation of the level above
    RowArgs pa;
    pa.vec_padded = true;
    const bool consumer_waits = (k + 1 < post) || (l > 0 && rows_can_push(LV[l - 1].P->S, pa));
    run_rows(h, W.d, W.A->S, last0 ? RowOp::SweepDot : RowOp::Sweep, a, s, (!last0 && consumer_waits) ? W.d : nullptr,
             t ? &h->ev_dom[h->dom_used] : nullptr);
    if (t) h->dom_used += 2;
    cur ^= 1;
  }
  if (level0 && post == 0)
    launch_dot(ctx, W.n, h->rz_weight ? h->rz_weight : b, W.x[cur], &h->red1, scal_mine(h, S_RZ), s);
  return W.x[cur];
}

double* vcycle_level(psc_hier* h, int l, const double* b, cudaStream_t s, bool timing, bool first_done = false) {
  return vcycle_rec(h, h->lv, l, b, s, timing, first_done, true);
}

// One Krylov iteration k >= 1, preconditioned by one V-cycle.
// PCG (P:113-117 with B = V-cycle; reading R1):
//   z = B r ; rz = (r, z) ; beta = rz / rz_old ; p = z + beta p ; rz_old = rz
//   q = A p ; pq = (p, q) ; alpha = rz_old / pq ; x += alpha p ; r -= alpha q ; rr = (r, r)
//   (at k = 1, p = 0 and rz_old = 1 so p = z exactly)
// FCG(1) (Notay): the same four reductions, fused the same way:
//   z = B r ; zq = (z, q_old) [last post-sweep] ; beta = zq / pq_old ; p = z - beta p ;
//   pr = (p, r) [same kernel] ; q = A p ; pq = (p, q) ; alpha = pr / pq ; x, r, rr as PCG
//   (at k = 1, q_old = 0 and pq_old = 1 so p = z exactly)
void record_iteration(psc_hier* h, cudaStream_t s, bool timing, int method) {
  psc_ctx* ctx = h->ctx;
  LevelWS& W = h->lv[0];
  const int R = ctx->nranks;
  const bool fcg = (method == PSC_KRYLOV_FCG);
  h->dom_used = 0;
  // the CG update of the previous iteration (or the eager start) wrote x_0 = M^{-1} r
  h->rz_weight = fcg ? h->q : nullptr;
  double* z = vcycle_level(h, 0, h->r_cg, s, timing);
  ctx->kt.level = -1;  // Krylov vector ops and q = A p
  h->rz_weight = nullptr;
  h->z_ptr = z;
  allgather_slot(h, S_RZ, s);
  if (fcg) {
    launch_fcg_dir(ctx, W.n, z, h->p, h->r_cg, scal(h, S_RZ), scal(h, S_PQ), R, &h->red1, scal_mine(h, S_PR), s);
    allgather_slot(h, S_PR, s);
  } else {
    launch_xpby(ctx, W.n, z, h->p, scal(h, S_RZ), rz_old(h), R, &h->red2, s);
  }
  {
    RowArgs a;
    a.vec_padded = true;  // library buffers, padded (dvec)
    a.x = h->p;
    a.y = h->q;
    a.red = &h->red1;
    a.red_out = scal_mine(h, S_PQ);
    prep(h, W.d, a, s);
    launch_rows(ctx, W.A->S, RowOp::SpmvDot, a, s);
    poison_halo(h, W.d, a.x, s);
  }
  allgather_slot(h, S_PQ, s);
  launch_cg_update(ctx, W.n, h->x_int, h->p, h->r_cg, h->q, scal(h, S_PQ), fcg ? scal(h, S_PR) : rz_old(h),
                   fcg ? R : 1, R, &h->red1, scal_mine(h, S_RR), s);
  allgather_slot(h, S_RR, s);
  PSC_CUDA(cudaMemcpyAsync(h->h_scal, h->d_scal, sizeof(double) * NSLOT * R, cudaMemcpyDeviceToHost, s));
}

void capture_iteration(psc_hier* h, int method, bool profile = false) {
  NvtxRange nv("psc_capture_iteration");
  psc_ctx* ctx = h->ctx;
  cudaStream_t s = ctx->stream;
  const int64_t l0 = ctx->launches, c0 = ctx->collectives;
  cudaGraph_t g = nullptr;
  const int dom_saved = h->dom_used;  // the timed solve graph's event pairs
  PSC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  if (profile) {
    ctx->kt.on = true;
    ctx->kt.recs.clear();
    ctx->kt.used = 0;
  }
  try {
    record_iteration(h, s, !profile, method);
    ctx->kt.on = false;
  } catch (...) {
    ctx->kt.on = false;
    h->rz_weight = nullptr;
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  PSC_CUDA(cudaStreamEndCapture(s, &g));
  cudaGraphExec_t& ex = profile ? h->prof_exec[method] : h->iter_exec[method];
  if (ex) PSC_CUDA(cudaGraphExecDestroy(ex));
  PSC_CUDA(cudaGraphInstantiate(&ex, g, 0));
  PSC_CUDA(cudaGraphDestroy(g));
  if (profile) {
    h->dom_used = dom_saved;
  } else {
    h->iter_launches[method] = ctx->launches - l0;
    h->iter_collectives[method] = ctx->collectives - c0;
  }
  ctx->launches = l0;
  ctx->collectives = c0;
}

double sum_ranks(const double* v, int R) {
  double s = 0.0;
  for (int r = 0; r < R; ++r) s += v[r];
  return s;
}

// Gather every rank's rows of a distributed matrix (host copies kept at
// psc_mat_create_csr for small matrices) and build a device layout of the whole
// matrix with global row and column numbering.
psc_mat* replicate_matrix(psc_ctx* ctx, psc_mat* A, int64_t n_rows_global, int64_t n_cols_global, bool allow_dia) {
  const int R = ctx->nranks;
  cudaStream_t s = ctx->stream;
  PSC_REQUIRE((int64_t)A->h_rowptr.size() == A->n_rows + 1, PSC_ERR_STATE, "replicated level matrix has no host copy");
  int64_t* dcnt = dalloc<int64_t>(2 * R + 2);
  int64_t mine[2] = {A->n_rows, A->nnz};
  PSC_CUDA(cudaMemcpy(dcnt + 2 * R, mine, sizeof(mine), cudaMemcpyHostToDevice));
  PSC_NCCL(ncclAllGather(dcnt + 2 * R, dcnt, 2, ncclInt64, ctx->comm, s));
  std::vector<int64_t> cnt(2 * R);
  PSC_CUDA(cudaMemcpyAsync(cnt.data(), dcnt, sizeof(int64_t) * 2 * R, cudaMemcpyDeviceToHost, s));
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(dcnt);
  int64_t totnnz = 0;
  for (int r = 0; r < R; ++r) totnnz += cnt[2 * r + 1];
  std::vector<int64_t> rp_all(n_rows_global + 1, 0), col_all(totnnz);
  std::vector<double> val_all(totnnz);
  int64_t row0 = 0, nz0 = 0;
  for (int r = 0; r < R; ++r) {
    const int64_t nr = cnt[2 * r], nz = cnt[2 * r + 1];
    int64_t* dp = dalloc<int64_t>(nr + 1 + nz);
    double* dv = dvec(nz);
    if (r == ctx->rank) {
      PSC_CUDA(cudaMemcpy(dp, A->h_rowptr.data(), sizeof(int64_t) * (nr + 1), cudaMemcpyHostToDevice));
      if (nz) {
        PSC_CUDA(cudaMemcpy(dp + nr + 1, A->h_colg.data(), sizeof(int64_t) * nz, cudaMemcpyHostToDevice));
        PSC_CUDA(cudaMemcpy(dv, A->h_val.data(), sizeof(double) * nz, cudaMemcpyHostToDevice));
      }
    }
    PSC_NCCL(ncclBroadcast(dp, dp, nr + 1 + nz, ncclInt64, r, ctx->comm, s));
    if (nz) PSC_NCCL(ncclBroadcast(dv, dv, nz, ncclDouble, r, ctx->comm, s));
    std::vector<int64_t> hp(nr + 1 + nz);
    PSC_CUDA(cudaMemcpyAsync(hp.data(), dp, sizeof(int64_t) * (nr + 1 + nz), cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaMemcpyAsync(val_all.data() + nz0, dv, sizeof(double) * nz, cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    dfree(dp);
    dfree(dv);
    for (int64_t i = 0; i < nr; ++i) rp_all[row0 + i + 1] = nz0 + hp[i + 1];
    std::copy(hp.begin() + nr + 1, hp.end(), col_all.begin() + nz0);
    row0 += nr;
    nz0 += nz;
  }
  PSC_REQUIRE(row0 == n_rows_global, PSC_ERR_STATE, "replicated rows do not add up");
  int64_t* drp = dalloc<int64_t>(n_rows_global + 1);
  int64_t* dcol = dalloc<int64_t>(totnnz);
  double* dval = dvec(totnnz);
  PSC_CUDA(cudaMemcpy(drp, rp_all.data(), sizeof(int64_t) * (n_rows_global + 1), cudaMemcpyHostToDevice));
  PSC_CUDA(cudaMemcpy(dcol, col_all.data(), sizeof(int64_t) * totnnz, cudaMemcpyHostToDevice));
  PSC_CUDA(cudaMemcpy(dval, val_all.data(), sizeof(double) * totnnz, cudaMemcpyHostToDevice));
  psc_mat* m = new psc_mat();
  m->ctx = ctx;
  m->n_rows = n_rows_global;
  m->nnz = totnnz;
  m->h_rowptr.swap(rp_all);  // host copy (AINV factors of the replicated levels)
  m->h_colg.swap(col_all);
  m->h_val.swap(val_all);
  try {
    sell_from_csr(ctx, n_rows_global, drp, dcol, dval, totnnz, 0, n_cols_global, nullptr, 0, m->S, s, 0, allow_dia);
  } catch (...) {
    dfree(drp);
    dfree(dcol);
    dfree(dval);
    delete m;
    throw;
  }
  m->assembled = true;
  dfree(drp);
  dfree(dcol);
  dfree(dval);
  return m;
}

// first replicated level: the first level >= 1 whose global size is at most
// PSC_REPL_ROWS (default 50000); -1 when none (or PSC_REPL_ROWS=0)
int replica_first(psc_hier* h) {
  if (h->ctx->nranks == 1 || h->L < 2) return -1;
  const char* e = getenv("PSC_REPL_ROWS");
  const int64_t lim = e ? atoll(e) : 50000;
  auto has_host = [&](int l) {  // every matrix of levels l.. has its host copy on this rank
    for (int k = l; k < h->L; ++k)
      for (psc_mat* m : {h->lv[k].A, h->lv[k].P, h->lv[k].R})
        if (m && (int64_t)m->h_rowptr.size() != m->n_rows + 1) return false;
    return true;
  };
  // Host copies are kept per rank by local size (api.cu), so the decision is agreed on
  // by all ranks: the replicated suffix is built only if every rank has the copies
  // (a rank-local choice would send ranks into different collectives).
  auto all_have_host = [&](int l) { return allreduce_min(h->ctx, has_host(l) ? 1 : 0) == 1; };
  for (int l = 1; l < h->L; ++l)
    if (h->lv[l].d->n_global <= lim) return all_have_host(l) ? l : -1;
  return (h->lv[h->L - 1].d->n_global <= coarse_smem_rows() && all_have_host(h->L - 1)) ? h->L - 1 : -1;
}

void level_coarse_solver(psc_hier* h, LevelWS& W) {
  W.one_cta = (W.nh == 0 && coarse_one_cta_fits(W.A->S));
  if (W.n <= coarse_dense_max_rows() && W.nh == 0 && !getenv("PSC_NO_DENSE_COARSE")) {
    W.dense = dvec(W.n * W.n + 1);
    dense_from_sell(h->ctx, W.A->S, W.dense, h->ctx->stream);
  }
}

// Dense suffix operator.  With the l1-Jacobi coarsest solver the V-cycle B_k of
// levels k.. (Eq. (2) applied recursively) is a fixed linear map;
// for the first level with at most PSC_DENSE_SUFFIX_ROWS rows (default 6144,
// 0 disables) it is precomputed column by column — the sub-cycle applied to the
// unit vectors — and each V-cycle then applies it as one dense product instead
// of the ~15 latency-bound launches of the deepest levels.  Same operator,
// different rounding order.  Not with PSC_COARSE_PCG (a nonlinear coarse solve).
void build_dense_suffix(psc_hier* h) {
  psc_ctx* ctx = h->ctx;
  if (h->opt.coarse_solver != PSC_COARSE_SWEEPS) return;
  const char* e = getenv("PSC_DENSE_SUFFIX_ROWS");
  const int64_t lim = std::min<int64_t>(e ? atoll(e) : 6144, dense_gemv_max_rows());
  if (lim <= 0) return;
  std::vector<LevelWS>* LV = nullptr;
  int k = -1;
  if (ctx->nranks == 1) {
    LV = &h->lv;
    for (int l = 1; l < h->L && k < 0; ++l)
      if (h->lv[l].n <= lim) k = l;
  } else if (h->rep.on) {
    LV = &h->rep.lv;
    for (int l = 0; l < (int)h->rep.lv.size() && k < 0; ++l)
      if (h->rep.lv[l].n <= lim) k = l;
  }
  if (k < 0) return;
  const bool dist = (LV == &h->lv);
  LevelWS& W = (*LV)[k];
  const int64_t n = W.n;
  cudaStream_t s = ctx->stream;
  double* DT = dvec(n * n);
  const double one = 1.0;
  for (int64_t j = 0; j < n; ++j) {
    PSC_CUDA(cudaMemsetAsync(W.b, 0, sizeof(double) * n, s));
    PSC_CUDA(cudaMemcpyAsync(W.b + j, &one, sizeof(double), cudaMemcpyHostToDevice, s));
    const double* xj = vcycle_rec(h, *LV, k, W.b, s, false, false, dist);
    PSC_CUDA(cudaMemcpyAsync(DT + j * n, xj, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }
  h->dsuf = dvec(n * n);
  launch_transpose(ctx, DT, n, h->dsuf, s);
  PSC_CUDA(cudaStreamSynchronize(s));
  dfree(DT);
  h->dsuf_lv = LV;
  h->dsuf_l = k;
}

void build_replica(psc_hier* h, int first) {
  psc_ctx* ctx = h->ctx;
  const int R = ctx->nranks;
  const int L = h->L;
  Replica& rp = h->rep;
  cudaStream_t s = ctx->stream;
  rp.first = first;
  rp.N = h->lv[first].d->n_global;
  for (int k = first; k < L; ++k) {
    LevelWS& D = h->lv[k];
    LevelWS W;
    W.n = D.d->n_global;
    W.A = replicate_matrix(ctx, D.A, W.n, W.n, true);
    rp.mats.push_back(W.A);
    if (k + 1 < L) {
      const int64_t nc = h->lv[k + 1].d->n_global;
      W.P = replicate_matrix(ctx, D.P, W.n, nc, false);
      W.R = replicate_matrix(ctx, D.R, nc, W.n, false);
      rp.mats.push_back(W.P);
      rp.mats.push_back(W.R);
    }
    W.dinv = dvec(W.n);
    launch_l1_dinv(ctx, W.A->S, W.dinv, s);
    for (double** b : {&W.x[0], &W.x[1], &W.r, &W.b}) {
      *b = dvec(W.n);
      PSC_CUDA(cudaMemsetAsync(*b, 0, sizeof(double) * W.n, s));
    }
    if (h->opt.smoother == PSC_SMOOTHER_AINV && k + 1 < L) build_ainv(h, W);
    if (k == L - 1) level_coarse_solver(h, W);
    rp.lv.push_back(W);
  }
  // b gather map: padded all-gather buffer (in the arena) -> global index; and
  // the owned+halo slots of level `first` -> global index
  LevelWS& W = h->lv[first];
  psc_desc* d = W.d;
  std::vector<int64_t> mf(rp.N);
  for (int r = 0; r < R; ++r)
    for (int64_t g = d->row_start[r]; g < d->row_start[r + 1]; ++g) mf[g] = r * rp.maxcnt + (g - d->row_start[r]);
  std::vector<int64_t> ml(W.n + W.nh);
  for (int64_t i = 0; i < W.n; ++i) ml[i] = d->own_begin + i;
  for (int64_t i = 0; i < W.nh; ++i) ml[W.n + i] = d->halo[i];
  rp.map_full = dalloc<int64_t>(rp.N);
  rp.map_loc = dalloc<int64_t>(ml.size());
  PSC_CUDA(cudaMemcpy(rp.map_full, mf.data(), sizeof(int64_t) * rp.N, cudaMemcpyHostToDevice));
  if (!ml.empty()) PSC_CUDA(cudaMemcpy(rp.map_loc, ml.data(), sizeof(int64_t) * ml.size(), cudaMemcpyHostToDevice));
  rp.sendbuf = dvec(rp.maxcnt);
  PSC_CUDA(cudaMemset(rp.sendbuf, 0, sizeof(double) * rp.maxcnt));
  PSC_CUDA(cudaStreamSynchronize(s));
  rp.on = true;
}

void free_hier(psc_hier* h) {
  if (!h) return;
  cudaSetDevice(h->ctx->device);
  if (h->ctx->stream) cudaStreamSynchronize(h->ctx->stream);
  p2p_free(h->ctx, h->p2p);
  for (auto& W : h->lv) {
    free_ainv(W);
    dfree(W.dinv);
    if (&W != &h->lv[0]) dfree(W.b);
    dfree(W.cz);
    dfree(W.cq);
  }
  Replica& rp = h->rep;
  for (auto& W : rp.lv) {
    free_ainv(W);
    dfree(W.dinv);
    dfree(W.x[0]);
    dfree(W.x[1]);
    dfree(W.r);
    dfree(W.b);
    dfree(W.dense);
    dfree(W.cz);
    dfree(W.cq);
  }
  for (psc_mat* m : rp.mats) {
    sell_free(m->S);
    delete m;
  }
  dfree(rp.sendbuf);
  dfree(rp.map_full);
  dfree(rp.map_loc);
  for (auto& W : h->lv) dfree(W.dense);
  dfree(h->r_cg);
  dfree(h->q);
  dfree(h->dsuf);
  dfree(h->arena);  // x[0], x[1], r of every level, x_int, p, d_scal, coarse gather buffer, flags
  dfree(h->d_bhost);
  dfree(h->d_xhost);
  if (h->h_scal) cudaFreeHost(h->h_scal);
  red_free(h->red1);
  red_free(h->red2);
  dfree(h->d_done);
  for (auto e : h->prof_exec)
    if (e) cudaGraphExecDestroy(e);
  for (auto e : h->iter_exec)
    if (e) cudaGraphExecDestroy(e);
  for (auto e : h->ev_dom) cudaEventDestroy(e);
  if (h->ev_t0) cudaEventDestroy(h->ev_t0);
  if (h->ev_t1) cudaEventDestroy(h->ev_t1);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  delete h;
}

// per-kernel sums of a profiled solve (psc_hier_kernel_profile)
struct KProf {
  std::vector<double> ms;  // per KTrace record of the iteration graph
  int iters = 0;
};

int solve_impl(psc_hier* h, int method, const double* b, double* x, double tol, int maxit, double* hist,
               psc_stats* st, double extra_h2d, KProf* prof = nullptr) {
  NvtxRange nv(method == PSC_KRYLOV_FCG ? "psc_fcg_solve" : "psc_pcg_solve");
  psc_ctx* ctx = h->ctx;
  cudaStream_t s = ctx->stream;
  const int R = ctx->nranks;
  LevelWS& W = h->lv[0];
  const int64_t l0 = ctx->launches, c0 = ctx->collectives;
  psc_stats S{};
  PSC_CUDA(cudaEventRecord(h->ev_t0, s));
  if (W.n) PSC_CUDA(cudaMemcpyAsync(h->x_int, x, sizeof(double) * W.n, cudaMemcpyDeviceToDevice, s));
  {
    RowArgs a;
    a.vec_padded = false;  // reads the caller's b
    a.x = h->x_int;
    a.b = b;
    a.y = h->r_cg;
    a.red = &h->red2;
    a.red_out = scal_mine(h, S_RR);
    a.red_stride = (int)((size_t)(S_BB - S_RR) * R);
    prep(h, W.d, a, s);
    launch_rows(ctx, W.A->S, RowOp::ResidDot2, a, s);
    poison_halo(h, W.d, a.x, s);
  }
  allgather_slot(h, S_RR, s);
  allgather_slot(h, S_BB, s);
  PSC_CUDA(cudaMemcpyAsync(h->h_scal, h->d_scal, sizeof(double) * NSLOT * R, cudaMemcpyDeviceToHost, s));
  PSC_CUDA(cudaStreamSynchronize(s));
  const double bb = sum_ranks(h->h_scal + S_BB * R, R);
  const double rr0 = sum_ranks(h->h_scal + S_RR * R, R);
  const double nb = std::sqrt(bb);
  int status = PSC_NOT_CONVERGED;
  int iters = 0;
  double rel = 0.0;
  double dom_ms = 0.0;
  int64_t dom_n = 0;
  if (nb == 0.0) {  // b = 0 -> x = 0 and no iteration
    if (W.n) PSC_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * W.n, s));
    status = PSC_OK;
    rel = 0.0;
    if (hist) hist[0] = 0.0;
  } else {
    rel = std::sqrt(rr0) / nb;
    if (hist) hist[0] = rel;
    if (rel <= tol) {
      status = PSC_OK;
    } else {
      PSC_CUDA(cudaMemsetAsync(h->p, 0, sizeof(double) * (W.n + W.nh), s));
      if (method == PSC_KRYLOV_FCG) {
        // q_old = 0 and pq_old = 1 (rank 0 holds the 1): p_1 = z_1 - 0 p_0 exactly
        PSC_CUDA(cudaMemsetAsync(h->q, 0, sizeof(double) * W.n, s));
        std::vector<double> pq0(R, 0.0);
        pq0[0] = 1.0;
        PSC_CUDA(cudaMemcpyAsync(scal(h, S_PQ), pq0.data(), sizeof(double) * R, cudaMemcpyHostToDevice, s));
      } else {
        const double one = 1.0;
        PSC_CUDA(cudaMemcpyAsync(rz_old(h), &one, sizeof(double), cudaMemcpyHostToDevice, s));
      }
      if (prof) {
        capture_iteration(h, method, true);
        prof->ms.assign(ctx->kt.recs.size(), 0.0);
      } else if (!h->iter_exec[method]) {
        capture_iteration(h, method);
      }
      cudaGraphExec_t ex = prof ? h->prof_exec[method] : h->iter_exec[method];
      for (int k = 1; k <= maxit; ++k) {
        PSC_CUDA(cudaGraphLaunch(ex, s));
        PSC_CUDA(cudaStreamSynchronize(s));
        if (prof) {
          for (size_t q = 0; q < ctx->kt.recs.size(); ++q) {
            float ms = 0.f;
            PSC_CUDA(cudaEventElapsedTime(&ms, ctx->kt.recs[q].e0, ctx->kt.recs[q].e1));
            prof->ms[q] += ms;
          }
          prof->iters = k;
        }
        ctx->launches += h->iter_launches[method];
        ctx->collectives += h->iter_collectives[method];
        for (int e = 0; e + 1 < h->dom_used; e += 2) {
          float ms = 0.f;
          PSC_CUDA(cudaEventElapsedTime(&ms, h->ev_dom[e], h->ev_dom[e + 1]));
          dom_ms += ms;
          dom_n++;
        }
        const double pq = sum_ranks(h->h_scal + S_PQ * R, R);
        const double rr = sum_ranks(h->h_scal + S_RR * R, R);
        iters = k;
        if (!(pq > 0.0) || !std::isfinite(pq)) {
          status = PSC_ERR_BREAKDOWN;
          break;
        }
        rel = std::sqrt(rr) / nb;
        if (hist) hist[k] = rel;
        if (rel <= tol) {
          status = PSC_OK;
          break;
        }
      }
    }
    if (W.n && status != PSC_ERR_BREAKDOWN)
      PSC_CUDA(cudaMemcpyAsync(x, h->x_int, sizeof(double) * W.n, cudaMemcpyDeviceToDevice, s));
  }
  PSC_CUDA(cudaEventRecord(h->ev_t1, s));
  PSC_CUDA(cudaStreamSynchronize(s));
  float tot = 0.f;
  PSC_CUDA(cudaEventElapsedTime(&tot, h->ev_t0, h->ev_t1));
  S.iters = iters;
  S.status = status;
  S.rel_res = rel;
  S.solve_seconds = tot * 1e-3;
  S.kernel_launches = ctx->launches - l0;
  S.collectives = ctx->collectives - c0;
  S.dom_kernel_seconds = dom_ms * 1e-3;
  S.dom_kernel_launches = dom_n;
  // bytes the level-0 sweep must move in its layout: 8 B per stored value, 4 B per
  // explicit column index (ELL slices), x in, b, dinv, x out
  S.dom_kernel_bytes = 8.0 * (double)W.A->nnz + 4.0 * (double)W.A->S.nnz_ell + 32.0 * (double)W.n;
  // level-0 sweep launches per iteration: pre-1 (the first pre-sweep from zero is
  // x = M^-1 b, no matrix) + post; one level: the coarsest solver's sweeps
  S.dom_kernel_per_iter = h->L > 1 ? std::max(h->opt.pre_sweeps - 1, 0) + h->opt.post_sweeps : 0;
  S.h2d_bytes = (int64_t)extra_h2d;
  S.halo_path = R == 1 ? 0 : (h->p2p.on ? 1 : 2);
  S.iter_graph_nodes = (int)h->iter_launches[method];
  if (st) *st = S;
  if (status == PSC_ERR_BREAKDOWN)
    throw Error(PSC_ERR_BREAKDOWN, method == PSC_KRYLOV_FCG ? "FCG breakdown: p^T A p <= 0 or not finite"
                                                            : "PCG breakdown: p^T A p <= 0 or not finite");
  return status;
}

}  // namespace

extern "C" {

int psc_hier_create(psc_ctx* ctx, int nlevels, psc_mat* const* A, psc_mat* const* P, psc_mat* const* R,
                    const psc_cycle_opts* opts, psc_hier** out) {
  NvtxRange nv("psc_hier_create");
  psc_hier* h = nullptr;
  try {
    PSC_REQUIRE(ctx && out && A && nlevels >= 1, PSC_ERR_ARG, "bad argument");
    PSC_REQUIRE(nlevels == 1 || (P && R), PSC_ERR_ARG, "P and R required for nlevels > 1");
    *out = nullptr;
    enter(ctx);
    h = new psc_hier();
    h->ctx = ctx;
    h->L = nlevels;
    if (opts) h->opt = *opts;
    PSC_REQUIRE(h->opt.pre_sweeps >= 0 && h->opt.post_sweeps >= 0 && h->opt.coarse_sweeps >= 0, PSC_ERR_ARG,
                "negative sweep count");
    PSC_REQUIRE(h->opt.coarse_solver == PSC_COARSE_SWEEPS || h->opt.coarse_solver == PSC_COARSE_PCG, PSC_ERR_ARG,
                "unknown coarse_solver");
    PSC_REQUIRE(h->opt.coarse_maxit >= 0 && h->opt.coarse_tol >= 0.0 && std::isfinite(h->opt.coarse_tol), PSC_ERR_ARG,
                "coarse_maxit / coarse_tol must be non-negative");
    PSC_REQUIRE(h->opt.variable_v == 0 || h->opt.variable_v == 1, PSC_ERR_ARG, "variable_v must be 0 or 1");
    PSC_REQUIRE(h->opt.smoother == PSC_SMOOTHER_L1JACOBI || h->opt.smoother == PSC_SMOOTHER_AINV, PSC_ERR_ARG,
                "unknown smoother");
    PSC_REQUIRE(h->opt.smoother != PSC_SMOOTHER_AINV || (h->opt.ainv_drop >= 0.0 && std::isfinite(h->opt.ainv_drop)),
                PSC_ERR_ARG, "ainv_drop must be a finite non-negative number");
    PSC_REQUIRE(!h->opt.variable_v || nlevels < 2 ||
                    (nlevels - 2 <= 20 && ((int64_t)std::max(h->opt.pre_sweeps, h->opt.post_sweeps) << (nlevels - 2)) <= (1 << 20)),
                PSC_ERR_ARG, "variable V-cycle: more than 2^20 sweeps at a level");
    if (h->opt.coarse_maxit == 0) h->opt.coarse_maxit = 40;
    if (h->opt.coarse_tol == 0.0) h->opt.coarse_tol = 1e-10;  // reading R23
    h->lv.resize(nlevels);
    for (int l = 0; l < nlevels; ++l) {
      LevelWS& W = h->lv[l];
      W.A = A[l];
      PSC_REQUIRE(W.A && W.A->assembled, PSC_ERR_STATE, "A_l missing or not assembled");
      PSC_REQUIRE(W.A->rows == W.A->cols, PSC_ERR_ARG, "A_l must map its index space to itself");
      W.d = W.A->rows;
      W.n = W.d->n_own;
      W.nh = W.d->n_halo();
      if (l + 1 < nlevels) {
        W.P = P[l];
        W.R = R[l];
        PSC_REQUIRE(W.P && W.R && W.P->assembled && W.R->assembled, PSC_ERR_STATE, "P_l/R_l missing or not assembled");
        PSC_REQUIRE(W.P->rows == W.d && W.P->cols == A[l + 1]->rows, PSC_ERR_ARG, "P_l: rows space l, cols space l+1");
        PSC_REQUIRE(W.R->rows == A[l + 1]->rows && W.R->cols == W.d, PSC_ERR_ARG, "R_l: rows space l+1, cols space l");
      }
    }
    cudaStream_t s = ctx->stream;
    const int NR = ctx->nranks;
    LevelWS& W0 = h->lv[0];
    // the arena: every buffer a peer writes into (halo-bearing vectors, gathered
    // scalars, the coarsest level's gather buffer, P2P flags), zero-initialised
    const int first = replica_first(h);
    psc_desc* dc = h->lv[first >= 0 ? first : nlevels - 1].d;
    int64_t maxcnt = 1;
    for (int r = 0; r < NR; ++r) maxcnt = std::max(maxcnt, dc->row_start[r + 1] - dc->row_start[r]);
    double* gbuf = nullptr;
    double* flagbuf = nullptr;
    std::vector<std::pair<double**, size_t>> plan;
    for (int l = 0; l < nlevels; ++l) {
      LevelWS& W = h->lv[l];
      for (double** b : {&W.x[0], &W.x[1], &W.r}) plan.push_back({b, (size_t)(W.n + W.nh) + 64});
    }
    plan.push_back({&h->x_int, (size_t)(W0.n + W0.nh) + 64});
    plan.push_back({&h->p, (size_t)(W0.n + W0.nh) + 64});
    plan.push_back({&h->d_scal, (size_t)NSLOT * NR + 1 + 64});
    if (NR > 1) plan.push_back({&gbuf, (size_t)NR * maxcnt + 64});
    plan.push_back({&flagbuf, (size_t)NR + 8});
    size_t total = 0;
    for (auto& pl : plan) total += (pl.second * sizeof(double) + 255) & ~(size_t)255;
    h->arena = dalloc<char>(total);
    PSC_CUDA(cudaMemset(h->arena, 0, total));
    size_t off = 0;
    for (auto& pl : plan) {
      *pl.first = reinterpret_cast<double*>(h->arena + off);
      off += (pl.second * sizeof(double) + 255) & ~(size_t)255;
    }
    for (int l = 0; l < nlevels; ++l) {
      LevelWS& W = h->lv[l];
      W.dinv = dvec(W.n);
      launch_l1_dinv(ctx, W.A->S, W.dinv, s);  // smoother build
      if (l > 0) W.b = dvec(W.n);
      if (h->opt.smoother == PSC_SMOOTHER_AINV && l + 1 < nlevels) build_ainv(h, W);
    }
    h->r_cg = dvec(W0.n);
    h->q = dvec(W0.n);
    W0.b = h->r_cg;
    if (NR > 1) {
      h->rep.gbuf = gbuf;
      h->rep.maxcnt = maxcnt;
    }
    PSC_CUDA(cudaMallocHost(&h->h_scal, sizeof(double) * ((size_t)NSLOT * ctx->nranks + 1)));
    h->red1 = red_alloc(ctx->num_sms, 1);
    h->red2 = red_alloc(ctx->num_sms, 2);
    h->d_done = dalloc<int>(1);
    PSC_CUDA(cudaMemset(h->d_done, 0, sizeof(int)));
    // live timing of the dominant kernel: one event pair around one level-0
    // sweep per iteration (each event-record node costs ~0.1% of an iteration);
    // PSC_DOM_TIMING=k times k of the 7 sweeps, 0 disables
    const char* dt = getenv("PSC_DOM_TIMING");
    const int nt = std::min(dt ? atoi(dt) : 1, std::max(h->opt.pre_sweeps - 1, 0) + h->opt.post_sweeps);
    const int ndom = 2 * std::max(nt, 0);
    h->ev_dom.resize(ndom);
    for (auto& e : h->ev_dom) PSC_CUDA(cudaEventCreate(&e));
    PSC_CUDA(cudaEventCreate(&h->ev_t0));
    PSC_CUDA(cudaEventCreate(&h->ev_t1));
    PSC_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    PSC_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    // coarsest solver: one CTA when the level is small enough; replicated on
    // every rank when distributed
    LevelWS& Wc = h->lv[nlevels - 1];
    if (ctx->nranks > 1) {
      if (first >= 0) build_replica(h, first);
      std::vector<P2PBufSpec> hb;
      std::vector<psc_desc*> ld;
      for (int l = 0; l < nlevels; ++l) {
        LevelWS& W = h->lv[l];
        ld.push_back(W.d);
        for (double* b : {W.x[0], W.x[1], W.r}) hb.push_back({b, l});
      }
      hb.push_back({h->x_int, 0});
      hb.push_back({h->p, 0});
      std::vector<P2PGatherSpec> gs;
      for (int sl = 0; sl < NSLOT; ++sl) gs.push_back({scal(h, (Slot)sl), ctx->rank});
      if (h->rep.on) gs.push_back({h->rep.gbuf, (int64_t)ctx->rank * h->rep.maxcnt});
      h->p2p.arena = h->arena;
      p2p_setup(ctx, h->p2p, hb, gs, ld, (char*)flagbuf - h->arena);
    } else {
      level_coarse_solver(h, Wc);
    }
    build_dense_suffix(h);
    if (h->opt.coarse_solver == PSC_COARSE_PCG) {  // buffers of the general coarsest PCG
      LevelWS& C = h->rep.on ? h->rep.lv.back() : Wc;
      if (!C.dense) {
        C.cz = dvec(C.n);
        C.cq = dvec(C.n);
      }
    }
    PSC_CUDA(cudaStreamSynchronize(s));
    *out = h;
    return PSC_OK;
  } catch (const Error& e) {
    free_hier(h);
    return hfail(ctx, e);
  } catch (const std::exception& e) {
    free_hier(h);
    return hfail(ctx, Error(PSC_ERR_ARG, e.what()));
  }
}

int psc_hier_info(psc_hier* h, int* nlevels, int64_t* n_owned, int64_t* nnz_A, int64_t* nnz_P, int64_t* nnz_R) {
  if (!h) return PSC_ERR_ARG;
  if (nlevels) *nlevels = h->L;
  for (int l = 0; l < h->L; ++l) {
    const LevelWS& W = h->lv[l];
    if (n_owned) n_owned[l] = W.n;
    if (nnz_A) nnz_A[l] = W.A->nnz;
    if (nnz_P) nnz_P[l] = W.P ? W.P->nnz : 0;
    if (nnz_R) nnz_R[l] = W.R ? W.R->nnz : 0;
  }
  return PSC_OK;
}

int psc_hier_vcycle(psc_hier* h, const double* r, double* z) {
  psc_ctx* ctx = h ? h->ctx : nullptr;
  try {
    PSC_REQUIRE(h && (r || h->lv[0].n == 0) && (z || h->lv[0].n == 0), PSC_ERR_ARG, "null argument");
    enter(ctx);
    cudaStream_t s = ctx->stream;
    LevelWS& W = h->lv[0];
    if (W.n) PSC_CUDA(cudaMemcpyAsync(h->r_cg, r, sizeof(double) * W.n, cudaMemcpyDeviceToDevice, s));
    double* zz = vcycle_level(h, 0, h->r_cg, s, false);
    if (W.n) PSC_CUDA(cudaMemcpyAsync(z, zz, sizeof(double) * W.n, cudaMemcpyDeviceToDevice, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    return PSC_OK;
  } catch (const Error& e) {
    return hfail(ctx, e);
  }
}

int psc_hier_dinv(psc_hier* h, int level, double* dinv) {
  psc_ctx* ctx = h ? h->ctx : nullptr;
  try {
    PSC_REQUIRE(h && level >= 0 && level < h->L, PSC_ERR_ARG, "bad level");
    enter(ctx);
    LevelWS& W = h->lv[level];
    if (W.n) PSC_CUDA(cudaMemcpyAsync(dinv, W.dinv, sizeof(double) * W.n, cudaMemcpyDeviceToDevice, ctx->stream));
    PSC_CUDA(cudaStreamSynchronize(ctx->stream));
    return PSC_OK;
  } catch (const Error& e) {
    return hfail(ctx, e);
  }
}

int psc_hier_smooth(psc_hier* h, int level, const double* b, double* x, int nsweeps) {
  psc_ctx* ctx = h ? h->ctx : nullptr;
  try {
    PSC_REQUIRE(h && level >= 0 && level < h->L && nsweeps >= 0, PSC_ERR_ARG, "bad argument");
    enter(ctx);
    cudaStream_t s = ctx->stream;
    LevelWS& W = h->lv[level];
    double* bl = W.b;
    if (W.n) PSC_CUDA(cudaMemcpyAsync(bl, b, sizeof(double) * W.n, cudaMemcpyDeviceToDevice, s));
    double* res;
    if (level == h->L - 1) res = coarse_sweeps(h, W, bl, nsweeps, s);
    else res = W.x[pre_smooth(h, W, bl, nsweeps, s, false)];
    if (W.n) PSC_CUDA(cudaMemcpyAsync(x, res, sizeof(double) * W.n, cudaMemcpyDeviceToDevice, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    return PSC_OK;
  } catch (const Error& e) {
    return hfail(ctx, e);
  }
}

int psc_hier_kernel_profile(psc_hier* h, int method, const double* b, int iters, psc_kernel_rec* recs, int max_recs,
                            int* n_recs) {
  psc_ctx* ctx = h ? h->ctx : nullptr;
  double* x = nullptr;
  try {
    PSC_REQUIRE(h && iters >= 1 && (b || h->lv[0].n == 0) && n_recs && (recs || max_recs == 0), PSC_ERR_ARG,
                "bad argument");
    PSC_REQUIRE(method == PSC_KRYLOV_PCG || method == PSC_KRYLOV_FCG, PSC_ERR_ARG, "unknown Krylov method");
    enter(ctx);
    x = dvec(h->lv[0].n + 1);
    PSC_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * (h->lv[0].n + 1), ctx->stream));
    KProf prof;
    solve_impl(h, method, b, x, 0.0, iters, nullptr, nullptr, 0.0, &prof);
    dfree(x);
    x = nullptr;
    // group the iteration's launches by (name, level), in order of first appearance
    std::vector<psc_kernel_rec> out;
    const auto& R = ctx->kt.recs;
    for (size_t q = 0; q < R.size(); ++q) {
      if (!R[q].name) continue;
      size_t o = 0;
      while (o < out.size() && !(out[o].level == R[q].level && std::strcmp(out[o].name, R[q].name) == 0)) ++o;
      if (o == out.size()) {
        psc_kernel_rec r{};
        std::snprintf(r.name, sizeof(r.name), "%s", R[q].name);
        r.level = R[q].level;
        out.push_back(r);
      }
      psc_kernel_rec& r = out[o];
      r.calls_per_iter += 1;
      r.total_us += 1e3 * prof.ms[q] / std::max(prof.iters, 1);
      r.alg_bytes += R[q].alg_bytes;
      r.layout_bytes += R[q].layout_bytes;
    }
    for (auto& r : out) {  // per call
      r.alg_bytes /= r.calls_per_iter;
      r.layout_bytes /= r.calls_per_iter;
    }
    *n_recs = (int)out.size();
    for (int q = 0; q < std::min<int>(max_recs, (int)out.size()); ++q) recs[q] = out[q];
    return PSC_OK;
  } catch (const Error& e) {
    dfree(x);
    return hfail(ctx, e);
  }
}

int psc_krylov_solve(psc_hier* h, int method, const double* b, double* x, double tol, int maxit, double* hist,
                     psc_stats* st) {
  psc_ctx* ctx = h ? h->ctx : nullptr;
  try {
    PSC_REQUIRE(h && maxit >= 0 && tol >= 0.0, PSC_ERR_ARG, "bad argument");
    PSC_REQUIRE(method == PSC_KRYLOV_PCG || method == PSC_KRYLOV_FCG, PSC_ERR_ARG, "unknown Krylov method");
    PSC_REQUIRE((b && x) || h->lv[0].n == 0, PSC_ERR_ARG, "null b/x");
    enter(ctx);
    return solve_impl(h, method, b, x, tol, maxit, hist, st, 0.0);
  } catch (const Error& e) {
    return hfail(ctx, e);
  }
}

int psc_pcg_solve(psc_hier* h, const double* b, double* x, double tol, int maxit, double* hist, psc_stats* st) {
  return psc_krylov_solve(h, PSC_KRYLOV_PCG, b, x, tol, maxit, hist, st);
}

int psc_pcg_solve_host(psc_hier* h, const double* b_host, double* x_host, double tol, int maxit, double* hist,
                       psc_stats* st) {
  return psc_krylov_solve_host(h, PSC_KRYLOV_PCG, b_host, x_host, tol, maxit, hist, st);
}

int psc_krylov_solve_host(psc_hier* h, int method, const double* b_host, double* x_host, double tol, int maxit,
                          double* hist, psc_stats* st) {
  psc_ctx* ctx = h ? h->ctx : nullptr;
  try {
    PSC_REQUIRE(h && maxit >= 0 && tol >= 0.0, PSC_ERR_ARG, "bad argument");
    PSC_REQUIRE(method == PSC_KRYLOV_PCG || method == PSC_KRYLOV_FCG, PSC_ERR_ARG, "unknown Krylov method");
    const int64_t n = h->lv[0].n;
    PSC_REQUIRE((b_host && x_host) || n == 0, PSC_ERR_ARG, "null b/x");
    enter(ctx);
    cudaStream_t s = ctx->stream;
    if (!h->d_bhost) {
      h->d_bhost = dvec(n);
      h->d_xhost = dvec(n);
    }
    if (n) {
      PSC_CUDA(cudaMemcpyAsync(h->d_bhost, b_host, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      PSC_CUDA(cudaMemcpyAsync(h->d_xhost, x_host, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    }
    psc_stats S{};
    int rc = solve_impl(h, method, h->d_bhost, h->d_xhost, tol, maxit, hist, &S, 16.0 * (double)n);
    if (n) PSC_CUDA(cudaMemcpyAsync(x_host, h->d_xhost, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    S.d2h_bytes = 8 * n;
    if (st) *st = S;
    return rc;
  } catch (const Error& e) {
    return hfail(ctx, e);
  }
}

int psc_hier_exchange_bench(psc_hier* h, int level, int reps, double* us_per_exchange) {
  psc_ctx* ctx = h ? h->ctx : nullptr;
  try {
    PSC_REQUIRE(h && level >= 0 && level < h->L && reps > 0 && us_per_exchange, PSC_ERR_ARG, "bad argument");
    enter(ctx);
    cudaStream_t s = ctx->stream;
    LevelWS& W = h->lv[level];
    for (int k = 0; k < 3; ++k) exchange(h, W.d, W.x[0], s);  // warm
    PSC_CUDA(cudaStreamSynchronize(s));
    PSC_CUDA(cudaEventRecord(h->ev_t0, s));
    for (int k = 0; k < reps; ++k) exchange(h, W.d, W.x[0], s);
    PSC_CUDA(cudaEventRecord(h->ev_t1, s));
    PSC_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    PSC_CUDA(cudaEventElapsedTime(&ms, h->ev_t0, h->ev_t1));
    *us_per_exchange = 1e3 * ms / reps;
    return PSC_OK;
  } catch (const Error& e) {
    return hfail(ctx, e);
  }
}

int psc_hier_rebuild_smoothers(psc_hier* h) {
  psc_ctx* ctx = h ? h->ctx : nullptr;
  try {
    PSC_REQUIRE(h, PSC_ERR_ARG, "null hierarchy");
    PSC_REQUIRE(!h->rep.on, PSC_ERR_STATE, "rebuild_smoothers: the replicated coarse suffix keeps its own copies");
    enter(ctx);
    cudaStream_t s = ctx->stream;
    PSC_CUDA(cudaStreamSynchronize(s));
    for (int l = 0; l < h->L; ++l) {
      LevelWS& W = h->lv[l];
      launch_l1_dinv(ctx, W.A->S, W.dinv, s);
      if (W.dense) dense_from_sell(ctx, W.A->S, W.dense, s);
      if (h->opt.smoother == PSC_SMOOTHER_AINV && l + 1 < h->L) build_ainv(h, W);
    }
    if (h->dsuf) {  // the dense suffix operator is a function of the smoothers
      dfree(h->dsuf);
      h->dsuf = nullptr;
      h->dsuf_lv = nullptr;
      h->dsuf_l = -1;
      build_dense_suffix(h);
    }
    // the captured iterations may hold buffers that were reallocated (AINV factors)
    for (auto& e : h->iter_exec)
      if (e) {
        PSC_CUDA(cudaGraphExecDestroy(e));
        e = nullptr;
      }
    for (auto& e : h->prof_exec)
      if (e) {
        PSC_CUDA(cudaGraphExecDestroy(e));
        e = nullptr;
      }
    PSC_CUDA(cudaStreamSynchronize(s));
    return PSC_OK;
  } catch (const Error& e) {
    return hfail(ctx, e);
  }
}

void psc_hier_destroy(psc_hier* h) { free_hier(h); }

}  // extern "C"
