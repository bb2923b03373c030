// pscgen.cpp — seeded input generator for the AMG-PCG solve phase.
//
// INPUT GENERATOR, NOT THE METHOD'S SOLVE PATH.  The north star (BASELINE.json)
// takes the aggregation hierarchy {A_l, P_l, R_l = P_l^T} as a *given* input;
// this file builds that input the way PSCToolkit's VBM set-up describes it, so
// that both the CUDA library (paper_2406_19754_b200/) and the CPU oracle
// (oracle/) can be fed the same matrices.  It contains none of the solve-phase
// arithmetic (no l1 diagonal, no smoothing sweep, no V-cycle, no CG); those live
// separately in the oracle and in the CUDA library and share no code.
//
// What is built (citations are PAPER.md line numbers + section):
//   * A_0: 7-point finite-difference 3D Poisson, -lap u = 1 on [0,1]^3 with
//     homogeneous Dirichlet boundary (Sec. 3), unscaled stencil
//     (6, -1) (reading R15); or the variable-coefficient diffusion of
//     BASELINE.json config 5 (reading R22).
//   * Row-block distribution by boxes: rank r owns a box of the grid and a
//     contiguous block of global rows (Sec. 2.1 "partitioning the index
//     space among processes"); numbering is rank-major, x-fastest in the box.
//   * Decoupled Vanek-Mandel-Brezina aggregation (Sec. 2.3.1): strong
//     set N_i(theta) = { j : |a_ij| >= theta sqrt(a_ii a_jj) }; aggregates never
//     cross a rank boundary ("decoupled").  Classical three phases (reading R18).
//   * Tentative prolongator Eq. (3) with near-kernel w = 1.
//   * Smoothed prolongator P = (I - omega D^-1 A) P^ with omega = 1/||D^-1 A||_inf
//     (P:240).
//   * Explicit restriction R = P^T (BASELINE.json north_star).
//   * Galerkin coarse operator A_{l+1} = P_l^T A_l P_l.
//
// Everything is computed for all ranks inside one process (logical ranks), with
// OpenMP over rows.  The global CSR of each level is the concatenation of the
// rank blocks, so rank r's piece is a contiguous row range.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>
#include <omp.h>
#include <cstdio>

#define PSC_GEN_CHECK(c)                                                               \
  do {                                                                                 \
    if (!(c)) {                                                                        \
      fprintf(stderr, "pscgen: check failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);  \
      abort();                                                                         \
    }                                                                                  \
  } while (0)

namespace {

template <class T>
struct Buf {  // uninitialised heap array (avoids zero-filling multi-GB vectors)
  std::unique_ptr<T[]> p;
  int64_t n = 0;
  void alloc(int64_t m) { p.reset(m ? new T[m] : nullptr); n = m; }
  T& operator[](int64_t i) { return p[i]; }
  const T& operator[](int64_t i) const { return p[i]; }
  T* data() { return p.get(); }
};

struct CSR {
  int64_t nrows = 0, ncols = 0;
  Buf<int64_t> ptr;  // nrows+1
  Buf<int64_t> col;  // nnz, strictly increasing per row
  Buf<double> val;   // nnz
  int64_t nnz() const { return nrows ? ptr[nrows] : 0; }
};

struct Level {
  int64_t n = 0;
  std::vector<int64_t> row_start;  // nranks+1
  CSR A, P, R;                     // P: n x n_next, R: n_next x n (absent at coarsest)
  std::vector<int64_t> agg;        // fine node -> global coarse id (absent at coarsest)
  std::vector<double> w, ph;       // matching: near-kernel vector of the level, tentative P^ values
};

struct Hier {
  int nranks = 1;
  std::vector<Level> lv;
  double omega_last = 0.0;
  std::vector<double> omega;  // per level (l < L-1)
};

// Chunked parallel CSR builder: rows [0, nrows) are cut into chunks; each chunk
// is filled by one thread into private vectors, then concatenated in row order.
struct ChunkOut {
  std::vector<int64_t> len;  // per row
  std::vector<int64_t> col;
  std::vector<double> val;
};

template <class RowFn>
void build_csr_chunked(CSR& out, int64_t nrows, int64_t ncols, RowFn&& row_fn) {
  const int64_t CH = 8192;
  const int64_t nch = (nrows + CH - 1) / CH;
  std::vector<ChunkOut> chunks(nch);
#pragma omp parallel
  {
    auto st = row_fn.make_state();
#pragma omp for schedule(dynamic, 1)
    for (int64_t c = 0; c < nch; ++c) {
      ChunkOut& co = chunks[c];
      const int64_t r0 = c * CH, r1 = std::min(nrows, r0 + CH);
      co.len.resize(r1 - r0);
      for (int64_t i = r0; i < r1; ++i) {
        size_t before = co.col.size();
        row_fn(st, i, co.col, co.val);
        co.len[i - r0] = (int64_t)(co.col.size() - before);
      }
    }
  }
  std::vector<int64_t> coff(nch + 1, 0);
  for (int64_t c = 0; c < nch; ++c) coff[c + 1] = coff[c] + (int64_t)chunks[c].col.size();
  out.nrows = nrows;
  out.ncols = ncols;
  out.ptr.alloc(nrows + 1);
  out.col.alloc(coff[nch]);
  out.val.alloc(coff[nch]);
  out.ptr[0] = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t c = 0; c < nch; ++c) {
    ChunkOut& co = chunks[c];
    const int64_t r0 = c * CH;
    int64_t o = coff[c];
    for (size_t k = 0; k < co.len.size(); ++k) {
      o += co.len[k];
      out.ptr[r0 + (int64_t)k + 1] = o;
    }
    std::memcpy(out.col.data() + coff[c], co.col.data(), co.col.size() * sizeof(int64_t));
    std::memcpy(out.val.data() + coff[c], co.val.data(), co.val.size() * sizeof(double));
    std::vector<int64_t>().swap(co.col);
    std::vector<double>().swap(co.val);
  }
}

// ---------------------------------------------------------------- A_0 (grid)
struct Grid {
  int64_t nx, ny, nz;  // global grid points
  int px, py, pz;      // process grid
  int64_t bx, by, bz;  // box per rank
  int64_t box_n() const { return bx * by * bz; }
  int64_t gidx(int64_t gx, int64_t gy, int64_t gz) const {
    int64_t rx = gx / bx, ry = gy / by, rz = gz / bz;
    int64_t r = rx + px * (ry + py * rz);
    int64_t lx = gx - rx * bx, ly = gy - ry * by, lz = gz - rz * bz;
    return r * box_n() + lx + bx * (ly + by * lz);
  }
  void coords(int64_t g, int64_t& gx, int64_t& gy, int64_t& gz) const {
    int64_t r = g / box_n(), li = g - r * box_n();
    int64_t rx = r % px, ry = (r / px) % py, rz = r / ((int64_t)px * py);
    int64_t lx = li % bx, ly = (li / bx) % by, lz = li / (bx * by);
    gx = rx * bx + lx;
    gy = ry * by + ly;
    gz = rz * bz + lz;
  }
};

// Variable-coefficient diffusion (reading R22): kappa = jump on a checkerboard
// of `cube`^3-cell cubes in global coordinates, else 1; face coefficient is the
// harmonic mean 2 k_i k_j/(k_i + k_j); a Dirichlet face contributes k_i.
struct Coef {
  int problem;  // 0 = Poisson, 1 = jump
  double jump;
  int64_t cube;
  double kappa(int64_t gx, int64_t gy, int64_t gz) const {
    if (problem == 0) return 1.0;
    int64_t s = gx / cube + gy / cube + gz / cube;
    return (s & 1) ? jump : 1.0;
  }
};

struct StencilRow {
  const Grid* g;
  const Coef* cf;
  int make_state() const { return 0; }
  void operator()(int&, int64_t i, std::vector<int64_t>& col, std::vector<double>& val) const {
    int64_t gx, gy, gz;
    g->coords(i, gx, gy, gz);
    const double ki = cf->kappa(gx, gy, gz);
    int64_t c[7];
    double v[7];
    int m = 0;
    double diag = 0.0;
    const int64_t d[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
    for (int f = 0; f < 6; ++f) {
      int64_t x = gx + d[f][0], y = gy + d[f][1], z = gz + d[f][2];
      if (x < 0 || y < 0 || z < 0 || x >= g->nx || y >= g->ny || z >= g->nz) {
        diag += ki;  // Dirichlet face
        continue;
      }
      double kj = cf->kappa(x, y, z);
      double t = (cf->problem == 0) ? 1.0 : 2.0 * ki * kj / (ki + kj);
      diag += t;
      c[m] = g->gidx(x, y, z);
      v[m] = -t;
      ++m;
    }
    c[m] = i;
    v[m] = diag;
    ++m;
    // insertion sort by column
    for (int a = 1; a < m; ++a) {
      int64_t cc = c[a];
      double vv = v[a];
      int b = a - 1;
      while (b >= 0 && c[b] > cc) { c[b + 1] = c[b]; v[b + 1] = v[b]; --b; }
      c[b + 1] = cc;
      v[b + 1] = vv;
    }
    for (int a = 0; a < m; ++a) { col.push_back(c[a]); val.push_back(v[a]); }
  }
};

// ------------------------------------------------------------- aggregation
// Decoupled VMB on one rank's block [r0, r1) of level matrix A (global CSR).
// Returns the number of aggregates; agg_local[i - r0] = local aggregate id.
int64_t vmb_aggregate_rank(const CSR& A, const double* diag, int64_t r0, int64_t r1, double theta,
                           int64_t* agg_local) {
  const int64_t nloc = r1 - r0;
  // strong sets (owned, j != i)
  std::vector<int64_t> sptr(nloc + 1, 0);
  std::vector<int64_t> sidx;
  std::vector<double> sstr;
  sidx.reserve((size_t)(A.ptr[r1] - A.ptr[r0]));
  sstr.reserve((size_t)(A.ptr[r1] - A.ptr[r0]));
  for (int64_t i = r0; i < r1; ++i) {
    for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      int64_t j = A.col[k];
      if (j == i || j < r0 || j >= r1) continue;
      double s = std::sqrt(diag[i] * diag[j]);
      double a = std::fabs(A.val[k]);
      if (a >= theta * s) {
        sidx.push_back(j - r0);
        sstr.push_back(a / s);
      }
    }
    sptr[i - r0 + 1] = (int64_t)sidx.size();
  }
  for (int64_t i = 0; i < nloc; ++i) agg_local[i] = -1;
  int64_t nagg = 0;
  // Phase 1: i and all its strong neighbours unaggregated -> new aggregate.
  for (int64_t i = 0; i < nloc; ++i) {
    if (agg_local[i] != -1) continue;
    bool free_nb = true;
    for (int64_t k = sptr[i]; k < sptr[i + 1]; ++k)
      if (agg_local[sidx[k]] != -1) { free_nb = false; break; }
    if (!free_nb) continue;
    agg_local[i] = nagg;
    for (int64_t k = sptr[i]; k < sptr[i + 1]; ++k) agg_local[sidx[k]] = nagg;
    ++nagg;
  }
  // Phase 2: join the phase-1 aggregate of the strongest strong neighbour
  // (snapshot of phase 1; ties -> lowest aggregate id).
  std::vector<int64_t> snap(agg_local, agg_local + nloc);
  for (int64_t i = 0; i < nloc; ++i) {
    if (snap[i] != -1) continue;
    double best = -1.0;
    int64_t bagg = -1;
    for (int64_t k = sptr[i]; k < sptr[i + 1]; ++k) {
      int64_t a = snap[sidx[k]];
      if (a == -1) continue;
      if (sstr[k] > best || (sstr[k] == best && a < bagg)) { best = sstr[k]; bagg = a; }
    }
    if (bagg != -1) agg_local[i] = bagg;
  }
  // Phase 3: leftovers form aggregates with their unaggregated strong neighbours.
  for (int64_t i = 0; i < nloc; ++i) {
    if (agg_local[i] != -1) continue;
    agg_local[i] = nagg;
    for (int64_t k = sptr[i]; k < sptr[i + 1]; ++k)
      if (agg_local[sidx[k]] == -1) agg_local[sidx[k]] = nagg;
    ++nagg;
  }
  return nagg;
}

// ------------------------------------------------- matching-based aggregation
// Coupled aggregation based on compatible weighted matching (Sec. 2.3.1;
// SPEC S:251-285), restricted to each rank's block here (reading R29):
//   edge weights c_ij = 1 - 2 a_ij w_i w_j / (a_ii w_i^2 + a_jj w_j^2) on the
//     off-diagonal pattern (usable when the denominator is non-zero and c_ij > 0);
//   approximate maximum weight matching: the locally dominant greedy -- repeatedly the
//     heaviest remaining edge (ties: lexicographically smallest (i, j)), its endpoints
//     removed (weight >= 1/2 of the optimum);
//   Eq. (4): a matched pair e = {i, j} gets the column w_e = (w_i, w_j) / ||(w_i, w_j)||,
//     an unmatched vertex s the column w_s / |w_s|; the coarse near-kernel vector is
//     P^_1^T w (||w_e|| for a pair, |w_s| for a singleton);
//   k sweeps ("aggregates of size 2^k"): sweep t matches the unsmoothed Galerkin
//     matrix of sweep t-1 and the composed P^ = P^_1 P^_2 ... P^_k has one entry per row.
// Returns the number of aggregates; agg[i] local aggregate, ph[i] = P^_{i, agg(i)}.
int64_t match_aggregate_rank(const CSR& A, int64_t r0, int64_t r1, const double* w0, int k, int64_t* agg_out,
                             double* ph_out) {
  const int64_t nloc = r1 - r0;
  // current level: local CSR (rows/cols 0..m-1), near-kernel vector
  std::vector<int64_t> ptr(nloc + 1, 0), col;
  std::vector<double> val, w(w0, w0 + nloc);
  for (int64_t i = r0; i < r1; ++i) {
    for (int64_t q = A.ptr[i]; q < A.ptr[i + 1]; ++q) {
      const int64_t j = A.col[q];
      if (j < r0 || j >= r1) continue;  // decoupled per rank block
      col.push_back(j - r0);
      val.push_back(A.val[q]);
    }
    ptr[i - r0 + 1] = (int64_t)col.size();
  }
  std::vector<int64_t> agg(nloc);
  std::vector<double> ph(nloc, 1.0);
  for (int64_t i = 0; i < nloc; ++i) agg[i] = i;
  int64_t m = nloc;
  for (int sweep = 0; sweep < k && m > 1; ++sweep) {
    std::vector<double> d(m, 0.0);
    for (int64_t i = 0; i < m; ++i)
      for (int64_t q = ptr[i]; q < ptr[i + 1]; ++q)
        if (col[q] == i) d[i] = val[q];
    struct Edge {
      double c;
      int64_t i, j;
    };
    std::vector<Edge> E;
    for (int64_t i = 0; i < m; ++i)
      for (int64_t q = ptr[i]; q < ptr[i + 1]; ++q) {
        const int64_t j = col[q];
        if (j <= i) continue;
        const double den = d[i] * w[i] * w[i] + d[j] * w[j] * w[j];
        if (den == 0.0) continue;
        const double c = 1.0 - 2.0 * val[q] * w[i] * w[j] / den;
        if (c > 0.0) E.push_back({c, i, j});
      }
    std::stable_sort(E.begin(), E.end(), [](const Edge& a, const Edge& b) {
      if (a.c != b.c) return a.c > b.c;
      if (a.i != b.i) return a.i < b.i;
      return a.j < b.j;
    });
    std::vector<int64_t> mate(m, -1);
    for (const Edge& e : E)
      if (mate[e.i] < 0 && mate[e.j] < 0) {
        mate[e.i] = e.j;
        mate[e.j] = e.i;
      }
    // coarse numbering in increasing index of each pair's (or singleton's) first node
    std::vector<int64_t> cid(m, -1);
    std::vector<double> cval(m), wc;
    int64_t mc = 0;
    for (int64_t i = 0; i < m; ++i) {
      if (cid[i] >= 0) continue;
      const int64_t j = mate[i];
      if (j < 0) {  // singleton: w_s / |w_s|, coarse w = |w_s|
        PSC_GEN_CHECK(w[i] != 0.0);
        cid[i] = mc;
        cval[i] = w[i] / std::fabs(w[i]);
        wc.push_back(std::fabs(w[i]));
      } else {  // pair: (w_i, w_j) / ||.||, coarse w = ||.||
        const double nrm = std::sqrt(w[i] * w[i] + w[j] * w[j]);
        PSC_GEN_CHECK(nrm != 0.0);
        cid[i] = cid[j] = mc;
        cval[i] = w[i] / nrm;
        cval[j] = w[j] / nrm;
        wc.push_back(nrm);
      }
      ++mc;
    }
    // compose the fine assignment and its value
    for (int64_t f = 0; f < nloc; ++f) {
      ph[f] *= cval[agg[f]];
      agg[f] = cid[agg[f]];
    }
    // unsmoothed Galerkin of this sweep: A_c[I, J] = sum cval_i a_ij cval_j
    std::vector<std::vector<std::pair<int64_t, double>>> rows(mc);
    for (int64_t i = 0; i < m; ++i)
      for (int64_t q = ptr[i]; q < ptr[i + 1]; ++q) {
        const int64_t j = col[q];
        rows[cid[i]].push_back({cid[j], cval[i] * val[q] * cval[j]});
      }
    std::vector<int64_t> nptr(mc + 1, 0), ncol;
    std::vector<double> nval;
    for (int64_t I = 0; I < mc; ++I) {
      auto& r = rows[I];
      std::stable_sort(r.begin(), r.end(), [](const std::pair<int64_t, double>& a,
                                              const std::pair<int64_t, double>& b) { return a.first < b.first; });
      for (size_t t = 0; t < r.size(); ++t) {
        if (!ncol.empty() && (int64_t)ncol.size() > nptr[I] && ncol.back() == r[t].first) nval.back() += r[t].second;
        else { ncol.push_back(r[t].first); nval.push_back(r[t].second); }
      }
      nptr[I + 1] = (int64_t)ncol.size();
    }
    ptr.swap(nptr);
    col.swap(ncol);
    val.swap(nval);
    w.swap(wc);
    m = mc;
  }
  for (int64_t f = 0; f < nloc; ++f) {
    agg_out[f] = agg[f];
    ph_out[f] = ph[f];
  }
  return m;
}

// ---------------------------------------------------------- prolongator
struct SmoothedPRow {
  const CSR* A;
  const double* diag;
  const int64_t* agg;
  double omega;
  bool smooth;
  const double* ph = nullptr;  // tentative value of each node (nullptr: 1, Eq. (3) with w = 1)
  int make_state() const { return 0; }
  void operator()(int&, int64_t i, std::vector<int64_t>& col, std::vector<double>& val) const {
    const double phi = ph ? ph[i] : 1.0;
    if (!smooth) {  // tentative prolongator: Eq. (3) with w = 1, or Eq. (4) (matching)
      col.push_back(agg[i]);
      val.push_back(phi);
      return;
    }
    // P_i. = P^_i. - (omega / a_ii) * sum_k a_ik P^_k.
    const int64_t k0 = A->ptr[i], k1 = A->ptr[i + 1];
    const size_t base = col.size();
    for (int64_t k = k0; k < k1; ++k) {
      int64_t J = agg[A->col[k]];
      double a = ph ? A->val[k] * ph[A->col[k]] : A->val[k];
      size_t t = base;
      while (t < col.size() && col[t] != J) ++t;
      if (t == col.size()) { col.push_back(J); val.push_back(a); }
      else val[t] += a;
    }
    const double s = omega / diag[i];
    bool have_own = false;
    for (size_t t = base; t < col.size(); ++t) {
      double v = -s * val[t];
      if (col[t] == agg[i]) { v = phi + v; have_own = true; }
      val[t] = v;
    }
    if (!have_own) { col.push_back(agg[i]); val.push_back(phi); }
    // sort the row by column
    const size_t m = col.size() - base;
    for (size_t a = 1; a < m; ++a) {
      int64_t cc = col[base + a];
      double vv = val[base + a];
      size_t b = a;
      while (b > 0 && col[base + b - 1] > cc) { col[base + b] = col[base + b - 1]; val[base + b] = val[base + b - 1]; --b; }
      col[base + b] = cc;
      val[base + b] = vv;
    }
  }
};

// R = P^T.  Parallel: column counts and slot claims with atomics, then every
// row of R is sorted by column, so the result is deterministic.
void transpose(const CSR& P, CSR& R) {
  const int64_t n = P.nrows, nc = P.ncols, nnz = P.nnz();
  R.nrows = nc;
  R.ncols = n;
  R.ptr.alloc(nc + 1);
  R.col.alloc(nnz);
  R.val.alloc(nnz);
  std::vector<int64_t> cnt(nc + 1, 0);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nnz; ++k) {
#pragma omp atomic
    cnt[P.col[k] + 1]++;
  }
  for (int64_t c = 0; c < nc; ++c) cnt[c + 1] += cnt[c];
  for (int64_t c = 0; c <= nc; ++c) R.ptr[c] = cnt[c];
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = P.ptr[i]; k < P.ptr[i + 1]; ++k) {
      const int64_t c = P.col[k];
      int64_t o;
#pragma omp atomic capture
      o = cnt[c]++;
      R.col[o] = i;
      R.val[o] = P.val[k];
    }
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t c = 0; c < nc; ++c) {
    const int64_t b = R.ptr[c], e = R.ptr[c + 1];
    for (int64_t x = b + 1; x < e; ++x) {  // insertion sort by row index (rows are short)
      const int64_t cc = R.col[x];
      const double vv = R.val[x];
      int64_t y = x - 1;
      while (y >= b && R.col[y] > cc) { R.col[y + 1] = R.col[y]; R.val[y + 1] = R.val[y]; --y; }
      R.col[y + 1] = cc;
      R.val[y + 1] = vv;
    }
  }
}

// Sparse product rows (Gustavson): C[i,:] = sum_k X[i,k] Y[k,:], accumulated in
// X's stored order, output columns sorted.  Used twice for the Galerkin
// operator A_{l+1} = R (A P): first AP = A P, then R (AP).
struct SpGEMMRow {
  const CSR *X, *Y;
  int64_t ncols;
  struct State {
    std::vector<double> acc;
    std::vector<int64_t> mark;
    std::vector<int64_t> touched;
  };
  State make_state() const {
    State s;
    s.acc.assign(ncols, 0.0);
    s.mark.assign(ncols, -1);
    return s;
  }
  void operator()(State& s, int64_t i, std::vector<int64_t>& col, std::vector<double>& val) const {
    s.touched.clear();
    for (int64_t a = X->ptr[i]; a < X->ptr[i + 1]; ++a) {
      const int64_t k = X->col[a];
      const double xv = X->val[a];
      for (int64_t c = Y->ptr[k]; c < Y->ptr[k + 1]; ++c) {
        const int64_t K = Y->col[c];
        if (s.mark[K] != i) { s.mark[K] = i; s.acc[K] = 0.0; s.touched.push_back(K); }
        s.acc[K] += xv * Y->val[c];
      }
    }
    std::sort(s.touched.begin(), s.touched.end());
    for (int64_t K : s.touched) { col.push_back(K); val.push_back(s.acc[K]); }
  }
};

// Galerkin rows A_c[J,:] = sum_i R[J,i] (AP)[i,:] with (AP)[i,:] = sum_k A[i,k] P[k,:]
// (the association R (A P) of SpGEMMRow, bit for bit: each (AP)[i,K] is summed in k
// order, then added to A_c[J,K] in i order) without storing AP: row i of AP is
// recomputed for every J that needs it (the stencil-like fine levels, where AP would
// be as large as A times the prolongator's row length).
struct RAPRow {
  const CSR *R, *A, *P;
  int64_t nc;
  struct State {
    std::vector<double> acc, acc2;
    std::vector<int64_t> mark, mark2;
    std::vector<int64_t> touched, touched2;
  };
  State make_state() const {
    State s;
    s.acc.assign(nc, 0.0);
    s.mark.assign(nc, -1);
    s.acc2.assign(nc, 0.0);
    s.mark2.assign(nc, -1);
    return s;
  }
  void operator()(State& s, int64_t J, std::vector<int64_t>& col, std::vector<double>& val) const {
    s.touched.clear();
    for (int64_t a = R->ptr[J]; a < R->ptr[J + 1]; ++a) {
      const int64_t i = R->col[a];
      const double rv = R->val[a];
      // row i of AP (mark2 keyed by the R entry a: unique per (J, i))
      s.touched2.clear();
      for (int64_t b = A->ptr[i]; b < A->ptr[i + 1]; ++b) {
        const int64_t k = A->col[b];
        const double av = A->val[b];
        for (int64_t c = P->ptr[k]; c < P->ptr[k + 1]; ++c) {
          const int64_t K = P->col[c];
          if (s.mark2[K] != a) { s.mark2[K] = a; s.acc2[K] = 0.0; s.touched2.push_back(K); }
          s.acc2[K] += av * P->val[c];
        }
      }
      for (int64_t K : s.touched2) {
        if (s.mark[K] != J) { s.mark[K] = J; s.acc[K] = 0.0; s.touched.push_back(K); }
        s.acc[K] += rv * s.acc2[K];
      }
    }
    std::sort(s.touched.begin(), s.touched.end());
    for (int64_t K : s.touched) { col.push_back(K); val.push_back(s.acc[K]); }
  }
};

struct Params {
  double theta = 0.01;
  int max_levels = 20;
  int64_t coarse_target = 200;
  double stall_ratio = 0.75;
  int smooth = 1;
  int aggr = 0;          // 0: decoupled VMB; 1: matching
  int match_sweeps = 3;  // matching: k sweeps, aggregates of at most 2^k nodes ("maximum size 8")
};

void diag_of(const CSR& A, std::vector<double>& d) {
  d.assign(A.nrows, 0.0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < A.nrows; ++i)
    for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
      if (A.col[k] == i) d[i] = A.val[k];
}

static bool verbose() { return getenv("PSCGEN_VERBOSE") != nullptr; }
#define TLOG(name)                                                                        \
  do {                                                                                    \
    if (verbose()) {                                                                      \
      double t1 = omp_get_wtime();                                                        \
      fprintf(stderr, "[pscgen] level %d %-12s %.2f s\n", l, name, t1 - t0);             \
      t0 = t1;                                                                            \
    }                                                                                     \
  } while (0)

void build_levels(Hier* h, const Params& prm) {
  for (;;) {
    double t0 = omp_get_wtime();
    Level& L = h->lv.back();
    const int l = (int)h->lv.size() - 1;
    if (L.n <= prm.coarse_target || l + 1 >= prm.max_levels) break;
    std::vector<double> diag;
    diag_of(L.A, diag);
    TLOG("diag");
    // decoupled aggregation, independently per rank
    std::vector<int64_t> agg_local(L.n);
    std::vector<int64_t> nagg(h->nranks);
    L.ph.clear();
    if (prm.aggr == 1) {
      // near-kernel vector w = 1 at level 0; at coarser levels P^_{l-1}^T w_{l-1} is
      // carried as the level's w (the unit vector's coarse image)
      if (L.w.empty()) L.w.assign(L.n, 1.0);
      L.ph.assign(L.n, 1.0);
#pragma omp parallel for schedule(dynamic, 1)
      for (int r = 0; r < h->nranks; ++r)
        nagg[r] = match_aggregate_rank(L.A, L.row_start[r], L.row_start[r + 1], L.w.data() + L.row_start[r],
                                       prm.match_sweeps, agg_local.data() + L.row_start[r],
                                       L.ph.data() + L.row_start[r]);
    } else {
#pragma omp parallel for schedule(dynamic, 1)
      for (int r = 0; r < h->nranks; ++r)
        nagg[r] = vmb_aggregate_rank(L.A, diag.data(), L.row_start[r], L.row_start[r + 1], prm.theta,
                                     agg_local.data() + L.row_start[r]);
    }
    TLOG("aggregate");
    std::vector<int64_t> crs(h->nranks + 1, 0);
    for (int r = 0; r < h->nranks; ++r) crs[r + 1] = crs[r] + nagg[r];
    const int64_t nc = crs[h->nranks];
    if ((double)nc > prm.stall_ratio * (double)L.n || nc >= L.n) break;
    L.agg.resize(L.n);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < h->nranks; ++r)
      for (int64_t i = L.row_start[r]; i < L.row_start[r + 1]; ++i) L.agg[i] = agg_local[i] + crs[r];
    std::vector<int64_t>().swap(agg_local);
    // omega = 1/||D^-1 A||_inf over the whole (global) matrix
    double nrm = 0.0;
#pragma omp parallel for reduction(max : nrm) schedule(static)
    for (int64_t i = 0; i < L.n; ++i) {
      double s = 0.0;
      for (int64_t k = L.A.ptr[i]; k < L.A.ptr[i + 1]; ++k) s += std::fabs(L.A.val[k]);
      s /= std::fabs(diag[i]);
      nrm = std::max(nrm, s);
    }
    const double omega = 1.0 / nrm;
    h->omega.push_back(prm.smooth ? omega : 0.0);
    SmoothedPRow prow{&L.A, diag.data(), L.agg.data(), omega, prm.smooth != 0,
                      L.ph.empty() ? nullptr : L.ph.data()};
    build_csr_chunked(L.P, L.n, nc, prow);
    TLOG("prolongator");
    transpose(L.P, L.R);
    TLOG("transpose");
    Level NL;
    NL.n = nc;
    NL.row_start = crs;
    if (prm.aggr == 1) {  // coarse near-kernel vector P^^T w: sum over each aggregate of ph_i w_i
      NL.w.assign(nc, 0.0);
      for (int64_t i = 0; i < L.n; ++i) NL.w[L.agg[i]] += L.ph[i] * L.w[i];
    }
    if (L.A.nnz() <= 8 * L.n) {  // stencil-like A: AP rows recomputed, not stored
      RAPRow rrow{&L.R, &L.A, &L.P, nc};
      build_csr_chunked(NL.A, nc, nc, rrow);
    } else {  // denser A: AP first, then R (AP)
      CSR AP;
      SpGEMMRow aprow{&L.A, &L.P, nc};
      build_csr_chunked(AP, L.n, nc, aprow);
      SpGEMMRow raprow{&L.R, &AP, nc};
      build_csr_chunked(NL.A, nc, nc, raprow);
    }
    TLOG("galerkin");
    h->lv.push_back(std::move(NL));
  }
}

}  // namespace

extern "C" {

// Build a hierarchy for the 7-point problem on an nx*ny*nz grid split into
// px*py*pz rank boxes.  problem: 0 = Poisson, 1 = jump diffusion.
void* pscgen_build_grid(int64_t nx, int64_t ny, int64_t nz, int px, int py, int pz, int problem,
                        double jump, int64_t cube, double theta, int max_levels, int64_t coarse_target,
                        double stall_ratio, int smooth, int aggr, int match_sweeps) {
  if (nx % px || ny % py || nz % pz) return nullptr;
  Grid g{nx, ny, nz, px, py, pz, nx / px, ny / py, nz / pz};
  Coef cf{problem, jump, cube};
  Hier* h = new Hier();
  h->nranks = px * py * pz;
  Level L0;
  L0.n = nx * ny * nz;
  L0.row_start.resize(h->nranks + 1);
  for (int r = 0; r <= h->nranks; ++r) L0.row_start[r] = (int64_t)r * g.box_n();
  StencilRow srow{&g, &cf};
  build_csr_chunked(L0.A, L0.n, L0.n, srow);
  h->lv.push_back(std::move(L0));
  Params prm;
  prm.theta = theta;
  prm.max_levels = max_levels;
  prm.coarse_target = coarse_target;
  prm.stall_ratio = stall_ratio;
  prm.smooth = smooth;
  prm.aggr = aggr;
  prm.match_sweeps = match_sweeps;
  build_levels(h, prm);
  return h;
}

// Build a hierarchy from a user-supplied global CSR A_0 (copied) and a
// contiguous row partition row_start[0..nranks].
void* pscgen_build_csr(int64_t n, const int64_t* ptr, const int64_t* col, const double* val, int nranks,
                       const int64_t* row_start, double theta, int max_levels, int64_t coarse_target,
                       double stall_ratio, int smooth, int aggr, int match_sweeps) {
  Hier* h = new Hier();
  h->nranks = nranks;
  Level L0;
  L0.n = n;
  L0.row_start.assign(row_start, row_start + nranks + 1);
  L0.A.nrows = n;
  L0.A.ncols = n;
  L0.A.ptr.alloc(n + 1);
  std::memcpy(L0.A.ptr.data(), ptr, (n + 1) * sizeof(int64_t));
  const int64_t nnz = ptr[n];
  L0.A.col.alloc(nnz);
  L0.A.val.alloc(nnz);
  std::memcpy(L0.A.col.data(), col, nnz * sizeof(int64_t));
  std::memcpy(L0.A.val.data(), val, nnz * sizeof(double));
  h->lv.push_back(std::move(L0));
  Params prm;
  prm.theta = theta;
  prm.max_levels = max_levels;
  prm.coarse_target = coarse_target;
  prm.stall_ratio = stall_ratio;
  prm.smooth = smooth;
  prm.aggr = aggr;
  prm.match_sweeps = match_sweeps;
  build_levels(h, prm);
  return h;
}

// One matching aggregation (k sweeps) of an n x n CSR with near-kernel vector w
// (tests: SPEC S:260-285 examples).  Returns the number of aggregates.
int64_t pscgen_match(int64_t n, const int64_t* ptr, const int64_t* col, const double* val, const double* w, int k,
                     int64_t* agg, double* ph) {
  CSR A;
  A.nrows = A.ncols = n;
  A.ptr.alloc(n + 1);
  std::memcpy(A.ptr.data(), ptr, (n + 1) * sizeof(int64_t));
  A.col.alloc(ptr[n]);
  A.val.alloc(ptr[n]);
  std::memcpy(A.col.data(), col, ptr[n] * sizeof(int64_t));
  std::memcpy(A.val.data(), val, ptr[n] * sizeof(double));
  return match_aggregate_rank(A, 0, n, w, k, agg, ph);
}

int pscgen_nlevels(void* hp) { return (int)((Hier*)hp)->lv.size(); }
int pscgen_nranks(void* hp) { return ((Hier*)hp)->nranks; }
int64_t pscgen_level_n(void* hp, int l) { return ((Hier*)hp)->lv[l].n; }
double pscgen_omega(void* hp, int l) { return ((Hier*)hp)->omega[l]; }
void pscgen_row_start(void* hp, int l, int64_t* out) {
  Level& L = ((Hier*)hp)->lv[l];
  std::copy(L.row_start.begin(), L.row_start.end(), out);
}
static CSR* pick(void* hp, int l, int kind) {
  Level& L = ((Hier*)hp)->lv[l];
  return kind == 0 ? &L.A : (kind == 1 ? &L.P : &L.R);
}
// kind: 0 = A_l, 1 = P_l, 2 = R_l.  Returns the global CSR arrays (borrowed).
int pscgen_csr(void* hp, int l, int kind, int64_t* nrows, int64_t* ncols, int64_t** ptr, int64_t** col,
               double** val) {
  Hier* h = (Hier*)hp;
  if (l < 0 || l >= (int)h->lv.size()) return -1;
  if (kind != 0 && l == (int)h->lv.size() - 1) return -1;
  CSR* m = pick(hp, l, kind);
  *nrows = m->nrows;
  *ncols = m->ncols;
  *ptr = m->ptr.data();
  *col = m->col.data();
  *val = m->val.data();
  return 0;
}
const int64_t* pscgen_agg(void* hp, int l) { return ((Hier*)hp)->lv[l].agg.data(); }
void pscgen_free(void* hp) { delete (Hier*)hp; }
void pscgen_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }

}  // extern "C"
