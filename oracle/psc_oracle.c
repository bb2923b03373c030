/* psc_oracle.c — CPU ORACLE for the AMG-PCG solve phase.  TEST INFRASTRUCTURE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this.  It shares no code with the CUDA library (paper_2406_19754_b200/): no
 * headers, no helpers, no constants.  Plain, slow, single-threaded, IEEE-754
 * binary64, compiled without fast-math and with -ffp-contract=off so every
 * a*b+c below is a rounded multiply followed by a rounded add.
 *
 * Every function follows PAPER.md (arXiv 2406.19754) step by step; `P:n` is a
 * PAPER.md line, with its section / equation.  Readings of silent or garbled
 * points are DESIGN.md §3 R1..R22.
 *
 * Matrices are global CSR (int64 row_ptr, int64 column, f64 value).  The
 * hierarchy {A_l, P_l, R_l} is GIVEN (BASELINE.json north_star).
 *
 * Threads (SURVEY.md §8(d) "Oracle timing"): the same source also builds with
 * -fopenmp (liboracle_omp.so, the cpu_baseline timed on all host cores).  Only
 * row-independent loops are parallel (each output element is computed by one
 * thread with the serial arithmetic), and dot products sum fixed 4096-element
 * chunks serially and then the chunk sums in chunk order (reading R13: any fixed
 * order), so both builds are bitwise identical for any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#define OR_PAR _Pragma("omp parallel for schedule(static)")
#else
#define OR_PAR
#endif

/* number of threads of the OpenMP build (1 in the serial build) */
int or_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

typedef struct {
  int64_t nrows, ncols;
  const int64_t* ptr;
  const int64_t* col;
  const double* val;
} or_csr;

typedef struct {
  int nlevels;      /* L: level 0 finest, L-1 coarsest */
  const or_csr* A;  /* A[0..L-1] */
  const or_csr* P;  /* P[0..L-2], n_l x n_{l+1} */
  const or_csr* R;  /* R[0..L-2], n_{l+1} x n_l, R_l = P_l^T given explicitly */
  int pre, post;    /* smoothing sweeps before/after the coarse correction (R4: 4 and 4) */
  int coarse;       /* l1-Jacobi sweeps at the coarsest level (30) */
  int coarse_pcg;   /* 1: coarsest solver = PCG with l1-Jacobi preconditioner (VBM) */
  int coarse_maxit; /* its iteration cap ("at most 40 iterations") */
  double coarse_tol;/* its relative-residual tolerance (reading R23) */
  int variable_v;   /* 1: variable V-cycle, pre/post sweeps doubled per level (P:330 footnote, R25) */
  int smoother;     /* 0: l1-Jacobi; 1: AINV (reading R27) on levels < L-1 */
  double ainv_drop; /* AINV drop tolerance */
  /* AINV blocks per level (block-Jacobi across ranks): ainv_nb[l] blocks with
   * row starts ainv_rs[l][0..nb]; NULL (or nb <= 1): the whole matrix */
  const int* ainv_nb;
  const int64_t* const* ainv_rs;
} or_hier;

int or_ainv(const or_csr* A, int nranks, const int64_t* row_start, double drop_tol, int64_t** zptr,
            int64_t** zrow, double** zval, double* p);

/* y = A x.  Row sums in stored column order. */
void or_spmv(const or_csr* A, const double* x, double* y) {
  OR_PAR
  for (int64_t i = 0; i < A->nrows; ++i) {
    double s = 0.0;
    for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k) s += A->val[k] * x[A->col[k]];
    y[i] = s;
  }
}

/* l1-Jacobi smoother matrix, P:269-272 (Sec. 2.3.2):
 *   M_l = diag(A_l) + diag( { sum_{j=1, j!=i}^{N} |a_ij| }_i )
 * over the whole row (reading R7).  m[i] is the i-th diagonal entry of M_l. */
void or_l1_diag(const or_csr* A, double* m) {
  OR_PAR
  for (int64_t i = 0; i < A->nrows; ++i) {
    double aii = 0.0, off = 0.0;
    for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k) {
      if (A->col[k] == i) aii = A->val[k];
      else off += fabs(A->val[k]);
    }
    m[i] = aii + off;
  }
}

/* One smoothing sweep x_new = x + M^{-1} (b - A x) (the factor (I - M^{-1}A)
 * of Eq. (2)), Jacobi: every row reads the old x (reading R8). */
void or_l1_sweep(const or_csr* A, const double* m, const double* b, const double* x, double* xnew) {
  OR_PAR
  for (int64_t i = 0; i < A->nrows; ++i) {
    double s = 0.0;
    for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k) s += A->val[k] * x[A->col[k]];
    xnew[i] = x[i] + (b[i] - s) / m[i];
  }
}

/* nsweeps sweeps starting from x = 0 (reading R6: smoothers start from zero).
 * Result in x.  work: n doubles. */
void or_l1_sweeps_from_zero(const or_csr* A, const double* m, const double* b, int nsweeps, double* x,
                            double* work) {
  const int64_t n = A->nrows;
  memset(x, 0, sizeof(double) * (size_t)n);
  for (int s = 0; s < nsweeps; ++s) {
    or_l1_sweep(A, m, b, x, work);
    memcpy(x, work, sizeof(double) * (size_t)n);
  }
}

static double* dalloc(int64_t n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

/* (a, b): serial sums over fixed chunks of 4096 entries, then the chunk sums in
 * chunk order (fixed order, independent of the thread count). */
static double dot(int64_t n, const double* a, const double* b) {
  const int64_t C = 4096, nc = (n + C - 1) / C;
  double* part = (double*)calloc((size_t)(nc > 0 ? nc : 1), sizeof(double));
  OR_PAR
  for (int64_t c = 0; c < nc; ++c) {
    double s = 0.0;
    const int64_t e = (c + 1) * C < n ? (c + 1) * C : n;
    for (int64_t i = c * C; i < e; ++i) s += a[i] * b[i];
    part[c] = s;
  }
  double s = 0.0;
  for (int64_t c = 0; c < nc; ++c) s += part[c];
  free(part);
  return s;
}

/* Coarsest solver of the paper's VBM configuration: "at most 40
 * iterations of the Preconditioned CG coupled to l1-Jacobi preconditioner".
 * PCG from x = 0 with M = diag(m) (m from or_l1_diag); stops after maxit
 * iterations or when ||r_k||_2 <= tol ||b||_2 (reading R23).  Returns the
 * number of iterations. */
int or_coarse_pcg(const or_csr* A, const double* m, const double* b, double* x, int maxit, double tol) {
  const int64_t n = A->nrows;
  double* r = dalloc(n);
  double* z = dalloc(n);
  double* p = dalloc(n);
  double* q = dalloc(n);
  memset(x, 0, sizeof(double) * (size_t)n);
  memcpy(r, b, sizeof(double) * (size_t)n);
  const double nb = sqrt(dot(n, b, b));
  int k = 0;
  if (nb > 0.0) {
    OR_PAR
    for (int64_t i = 0; i < n; ++i) z[i] = r[i] / m[i];
    memcpy(p, z, sizeof(double) * (size_t)n);
    double rz = dot(n, r, z);
    for (k = 1; k <= maxit; ++k) {
      or_spmv(A, p, q);
      const double pq = dot(n, p, q);
      if (!(pq > 0.0)) { k -= 1; break; }
      const double alpha = rz / pq;
      OR_PAR
      for (int64_t i = 0; i < n; ++i) x[i] = x[i] + alpha * p[i];
      OR_PAR
      for (int64_t i = 0; i < n; ++i) r[i] = r[i] - alpha * q[i];
      if (sqrt(dot(n, r, r)) <= tol * nb) break;
      OR_PAR
      for (int64_t i = 0; i < n; ++i) z[i] = r[i] / m[i];
      const double rz_new = dot(n, r, z);
      const double beta = rz_new / rz;
      rz = rz_new;
      OR_PAR
      for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
    if (k > maxit) k = maxit;
  }
  free(r); free(z); free(p); free(q);
  return k;
}

/* Smoother of one level: l1-Jacobi (m) or AINV (Z by columns, pivots p). */
typedef struct {
  double* m;
  int64_t *zp, *zr;
  double *zv, *p;
} or_smoother;

/* x_new = x + M^-1 (b - A x) with the level's smoother (Eq. (2) factor I - M^-1 A);
 * AINV: M^-1 = Z D^-1 Z^T, D = diag(p) (reading R27) */
static void smooth_sweep(const or_hier* h, const or_smoother* sm, const or_csr* A, const double* b, const double* x,
                         double* xnew) {
  const int64_t n = A->nrows;
  if (!h->smoother) {
    or_l1_sweep(A, sm->m, b, x, xnew);
    return;
  }
  double* r = dalloc(n);
  double* u = dalloc(n);
  or_spmv(A, x, r);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  for (int64_t j = 0; j < n; ++j) { /* u = D^-1 Z^T r */
    double t = 0.0;
    for (int64_t q = sm->zp[j]; q < sm->zp[j + 1]; ++q) t += sm->zv[q] * r[sm->zr[q]];
    u[j] = t / sm->p[j];
  }
  for (int64_t k = 0; k < n; ++k) xnew[k] = 0.0; /* Z u, column by column */
  for (int64_t j = 0; j < n; ++j)
    for (int64_t q = sm->zp[j]; q < sm->zp[j + 1]; ++q) xnew[sm->zr[q]] += sm->zv[q] * u[j];
  for (int64_t k = 0; k < n; ++k) xnew[k] = x[k] + xnew[k];
  free(r); free(u);
}

/* nsweeps smoothing sweeps from x = 0 (reading R6) */
static void smooth_from_zero(const or_hier* h, const or_smoother* sm, const or_csr* A, const double* b, int nsweeps,
                             double* x) {
  const int64_t n = A->nrows;
  double* w = dalloc(n);
  memset(x, 0, sizeof(double) * (size_t)n);
  for (int s = 0; s < nsweeps; ++s) {
    smooth_sweep(h, sm, A, b, x, w);
    memcpy(x, w, sizeof(double) * (size_t)n);
  }
  free(w);
}

/* x = B_l b, the V-cycle of Eq. (2) (Sec. 2.3):
 *   I - B_l A_l = (I - M_l^{-T} A_l)(I - P_l B_{l+1} P_l^T A_l)(I - M_l^{-1} A_l),
 * applied to b with x = 0 on entry, i.e. right to left:
 *   pre:    x <- x + M^{-1}(b - A x), `pre` times                 (rightmost factor)
 *   coarse: x <- x + P B_{l+1} R (b - A x), R = P^T              (middle factor)
 *   post:   x <- x + M^{-T}(b - A x), `post` times; M diagonal so M^{-T} = M^{-1} (R9)
 * and B_ell at the coarsest level = `coarse` sweeps from zero. */
static void vcycle_level(const or_hier* h, const or_smoother* sm, int l, const double* b, double* x) {
  const or_csr* A = &h->A[l];
  const int64_t n = A->nrows;
  double* w = dalloc(n);
  if (l == h->nlevels - 1) {
    if (h->coarse_pcg) or_coarse_pcg(A, sm[l].m, b, x, h->coarse_maxit, h->coarse_tol);
    else or_l1_sweeps_from_zero(A, sm[l].m, b, h->coarse, x, w);
    free(w);
    return;
  }
  /* variable V-cycle (VMATCH, P:330 footnote): "2 smoother iteration at the
   * first level, and doubled at each following level" -> pre/post sweeps at
   * level l = pre/post * 2^l (reading R25: both pre and post double) */
  const int pre = h->variable_v ? h->pre << l : h->pre;
  const int post = h->variable_v ? h->post << l : h->post;
  smooth_from_zero(h, &sm[l], A, b, pre, x);
  /* coarse-grid correction */
  const or_csr* R = &h->R[l];
  const or_csr* P = &h->P[l];
  const int64_t nc = R->nrows;
  double* r = dalloc(n);
  double* bc = dalloc(nc);
  double* xc = dalloc(nc);
  or_spmv(A, x, r);
  OR_PAR
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  or_spmv(R, r, bc);
  vcycle_level(h, sm, l + 1, bc, xc);
  or_spmv(P, xc, r);
  OR_PAR
  for (int64_t i = 0; i < n; ++i) x[i] = x[i] + r[i];
  free(r);
  free(bc);
  free(xc);
  for (int s = 0; s < post; ++s) {
    smooth_sweep(h, &sm[l], A, b, x, w);
    memcpy(x, w, sizeof(double) * (size_t)n);
  }
  free(w);
}

/* the smoothers of every level: l1 diagonal (all levels: also the coarsest solver's),
 * and AINV factors of the levels < L-1 when h->smoother == 1 (block of one rank) */
static or_smoother* make_m(const or_hier* h) {
  or_smoother* sm = (or_smoother*)calloc((size_t)h->nlevels, sizeof(or_smoother));
  for (int l = 0; l < h->nlevels; ++l) {
    sm[l].m = dalloc(h->A[l].nrows);
    or_l1_diag(&h->A[l], sm[l].m);
    if (h->smoother == 1 && l < h->nlevels - 1) {
      const int64_t whole[2] = {0, h->A[l].nrows};
      const int blocked = h->ainv_nb && h->ainv_rs && h->ainv_nb[l] > 1 && h->ainv_rs[l];
      sm[l].p = dalloc(h->A[l].nrows);
      or_ainv(&h->A[l], blocked ? h->ainv_nb[l] : 1, blocked ? h->ainv_rs[l] : whole, h->ainv_drop, &sm[l].zp,
              &sm[l].zr, &sm[l].zv, sm[l].p);
    }
  }
  return sm;
}
static void free_m(const or_hier* h, or_smoother* sm) {
  for (int l = 0; l < h->nlevels; ++l) {
    free(sm[l].m); free(sm[l].zp); free(sm[l].zr); free(sm[l].zv); free(sm[l].p);
  }
  free(sm);
}

/* z = B_0 r (one V-cycle from x = 0). */
void or_vcycle(const or_hier* h, const double* r, double* z) {
  or_smoother* m = make_m(h);
  vcycle_level(h, m, 0, r, z);
  free_m(h, m);
}

/* Preconditioned CG (reading R1: PCG, equal to FCG(1) for a fixed SPD B;
 * P:113-117) with B = one V-cycle per iteration.
 * Stopping rule hist[k] = ||r_k||_2/||b||_2 <= tol on the recurrence residual
 * (reading R2).  x holds x_0 on entry (Fig. 6 caption), the solution on exit.
 * hist: maxit+1 doubles.  Returns 0 converged, 1 not converged, -6 breakdown
 * (p^T A p <= 0 or not finite).  *iters = iterations performed. */
int or_pcg(const or_hier* h, const double* b, double* x, double tol, int maxit, double* hist, int* iters) {
  const or_csr* A = &h->A[0];
  const int64_t n = A->nrows;
  *iters = 0;
  const double nb = sqrt(dot(n, b, b));
  if (nb == 0.0) { /* b = 0 -> x = 0, no iterations (R10) */
    memset(x, 0, sizeof(double) * (size_t)n);
    hist[0] = 0.0;
    return 0;
  }
  or_smoother* m = make_m(h);
  double* r = dalloc(n);
  double* z = dalloc(n);
  double* p = dalloc(n);
  double* q = dalloc(n);
  int status = 1;
  or_spmv(A, x, r);
  OR_PAR
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  hist[0] = sqrt(dot(n, r, r)) / nb;
  if (hist[0] <= tol) { status = 0; goto done; }
  vcycle_level(h, m, 0, r, z);
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rz = dot(n, r, z);
  for (int k = 1; k <= maxit; ++k) {
    or_spmv(A, p, q);
    const double pq = dot(n, p, q);
    if (!(pq > 0.0) || !isfinite(pq)) { status = -6; *iters = k; goto done; }
    const double alpha = rz / pq;
    OR_PAR
    for (int64_t i = 0; i < n; ++i) x[i] = x[i] + alpha * p[i];
    OR_PAR
    for (int64_t i = 0; i < n; ++i) r[i] = r[i] - alpha * q[i];
    hist[k] = sqrt(dot(n, r, r)) / nb;
    *iters = k;
    if (hist[k] <= tol) { status = 0; goto done; }
    vcycle_level(h, m, 0, r, z);
    const double rz_new = dot(n, r, z);
    const double beta = rz_new / rz;
    rz = rz_new;
    OR_PAR
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
done:
  free(r); free(z); free(p); free(q);
  free_m(h, m);
  return status;
}

/* Flexible CG, FCG(1) of Notay (the paper's Krylov method, Fig. 6;
 * its reference [MR1797890]): the preconditioner may vary between iterations
 * (e.g. the coarsest PCG solve makes B nonlinear), so each new direction is
 * explicitly A-orthogonalised against the previous one:
 *   z_k = B(r_k);  p_k = z_k - ((z_k, A p_{k-1}) / (p_{k-1}, A p_{k-1})) p_{k-1}
 *   alpha_k = (p_k, r_k) / (p_k, A p_k);  x += alpha_k p_k;  r -= alpha_k A p_k
 * Same stopping rule, history and status codes as or_pcg. */
int or_fcg(const or_hier* h, const double* b, double* x, double tol, int maxit, double* hist, int* iters) {
  const or_csr* A = &h->A[0];
  const int64_t n = A->nrows;
  *iters = 0;
  const double nb = sqrt(dot(n, b, b));
  if (nb == 0.0) {
    memset(x, 0, sizeof(double) * (size_t)n);
    hist[0] = 0.0;
    return 0;
  }
  or_smoother* m = make_m(h);
  double* r = dalloc(n);
  double* z = dalloc(n);
  double* p = dalloc(n);
  double* q = dalloc(n);
  int status = 1;
  double delta = 0.0;
  or_spmv(A, x, r);
  OR_PAR
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  hist[0] = sqrt(dot(n, r, r)) / nb;
  if (hist[0] <= tol) { status = 0; goto done; }
  for (int k = 1; k <= maxit; ++k) {
    vcycle_level(h, m, 0, r, z);
    if (k == 1) {
      memcpy(p, z, sizeof(double) * (size_t)n);
    } else {
      const double beta = dot(n, z, q) / delta; /* q = A p_{k-1} */
      OR_PAR
      for (int64_t i = 0; i < n; ++i) p[i] = z[i] - beta * p[i];
    }
    or_spmv(A, p, q);
    delta = dot(n, p, q);
    if (!(delta > 0.0) || !isfinite(delta)) { status = -6; *iters = k; goto done; }
    const double alpha = dot(n, p, r) / delta;
    OR_PAR
    for (int64_t i = 0; i < n; ++i) x[i] = x[i] + alpha * p[i];
    OR_PAR
    for (int64_t i = 0; i < n; ++i) r[i] = r[i] - alpha * q[i];
    hist[k] = sqrt(dot(n, r, r)) / nb;
    *iters = k;
    if (hist[k] <= tol) { status = 0; goto done; }
  }
done:
  free(r); free(z); free(p); free(q);
  free_m(h, m);
  return status;
}

/* ======================================================================
 * NEXT-1: the set-up the paper runs before the solve:
 * decoupled Vanek-Mandel-Brezina aggregation (Sec. 2.3.1), the
 * tentative prolongator of Eq. (3) with w = 1, its smoothing
 * P = (I - omega D^-1 A) P^ with omega = 1/||D^-1 A||_inf, R = P^T and
 * the Galerkin product A_{l+1} = P_l^T A_l P_l.  Readings: DESIGN.md
 * R17-R21 (theta, phases, stop rule, decoupling, omega) and R26 (phase 1 visits the
 * nodes in increasing global index).  Outputs are malloc'd CSR arrays the
 * caller frees with or_free.
 * ====================================================================== */

void or_free(void* p) { free(p); }

/* Decoupled VMB aggregation of A (square, global CSR) over the row blocks
 * row_start[0..nranks]: aggregates never contain nodes of two blocks (P:214,
 * "Decoupled"; strong couplings to another block are ignored).
 *   strong(i, j): j != i, same block, |a_ij| >= theta sqrt(a_ii a_jj)
 *   phase 1: visit the nodes in increasing global index (reading R26); i becomes a
 *            root when neither i nor any strong neighbour of i is aggregated yet; its
 *            aggregate is i and its strong neighbours (the VMB root rule)
 *   numbering: aggregate ids = roots in increasing global index (block by block)
 *   phase 2: "any remaining nodes are added to the nearest aggregates":
 *            a node outside the phase-1 aggregates joins the phase-1 aggregate of its
 *            strongest strong neighbour (largest |a_ij| / sqrt(a_ii a_jj)) that is in
 *            one; ties go to the lowest aggregate id (reading R18)
 *   phase 3: a node still unaggregated would start its own aggregate; this never
 *            happens, because phase 1 leaves no node farther than two strong edges
 *            from a root.
 * agg[n]: aggregate of each node; root[n]: 1 for roots.  Returns the number of
 * aggregates, or -1 if phase 3 was reached. */
int64_t or_vmb_aggregate(const or_csr* A, int nranks, const int64_t* row_start, double theta, int64_t* agg,
                         int8_t* root) {
  const int64_t n = A->nrows;
  double* d = dalloc(n);
  int64_t* blk = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  for (int r = 0; r < nranks; ++r)
    for (int64_t i = row_start[r]; i < row_start[r + 1]; ++i) blk[i] = r;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k)
      if (A->col[k] == i) d[i] = A->val[k];
  /* strong flags per stored entry */
  int8_t* st = (int8_t*)calloc((size_t)(A->ptr[n] > 0 ? A->ptr[n] : 1), 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k) {
      const int64_t j = A->col[k];
      st[k] = (j != i && blk[j] == blk[i] && fabs(A->val[k]) >= theta * sqrt(d[i] * d[j])) ? 1 : 0;
    }
  int8_t* in1 = (int8_t*)calloc((size_t)(n > 0 ? n : 1), 1); /* aggregated in phase 1 */
  int64_t* owner = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1)); /* root of the phase-1 aggregate */
  for (int64_t i = 0; i < n; ++i) { /* phase 1 */
    root[i] = 0;
    if (in1[i]) continue;
    int free_nb = 1;
    for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k)
      if (st[k] && in1[A->col[k]]) { free_nb = 0; break; }
    if (!free_nb) continue;
    root[i] = 1;
    in1[i] = 1;
    owner[i] = i;
    for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k)
      if (st[k]) { in1[A->col[k]] = 1; owner[A->col[k]] = i; }
  }
  /* aggregate ids: roots in increasing index */
  int64_t* rid = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t nc = 0;
  for (int64_t i = 0; i < n; ++i) rid[i] = root[i] ? nc++ : -1;
  for (int64_t i = 0; i < n; ++i) agg[i] = in1[i] ? rid[owner[i]] : -1;
  /* phase 2 from the phase-1 snapshot */
  int64_t left = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (in1[i]) continue;
    double best = -1.0;
    int64_t ba = -1;
    for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k) {
      const int64_t j = A->col[k];
      if (!st[k] || !in1[j]) continue;
      const double s = fabs(A->val[k]) / sqrt(d[i] * d[j]);
      const int64_t a = rid[owner[j]];
      if (s > best || (s == best && a < ba)) { best = s; ba = a; }
    }
    agg[i] = ba;
    if (ba < 0) ++left;
  }
  free(d); free(blk); free(st); free(in1); free(owner); free(rid);
  return left ? -1 : nc;
}

/* omega = 1 / ||D^-1 A||_inf = 1 / max_i sum_j |a_ij| / |a_ii|   (reading R21) */
double or_omega(const or_csr* A) {
  double mx = 0.0;
  for (int64_t i = 0; i < A->nrows; ++i) {
    double s = 0.0, dii = 0.0;
    for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k) {
      s += fabs(A->val[k]);
      if (A->col[k] == i) dii = A->val[k];
    }
    const double t = s / fabs(dii);
    if (t > mx) mx = t;
  }
  return 1.0 / mx;
}

/* Smoothed prolongator P = (I - omega D^-1 A) P^ with the tentative P^ of
 * Eq. (3), w = 1: P^_{iJ} = 1 if i in C_J.  Row i:
 *   t_J = sum_{k in row i, agg(k) = J} a_ik (stored column order),  s = omega / a_ii,
 *   P_iJ = 1 - s t_J if J = agg(i), else -s t_J;  one entry per aggregate J touched
 * by row i, columns increasing.  Outputs malloc'd (ptr[n+1], col, val). */
void or_smoothed_prolongator(const or_csr* A, const int64_t* agg, int64_t nc, double omega, int64_t** pptr,
                             int64_t** pcol, double** pval) {
  const int64_t n = A->nrows;
  int64_t* ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* col = (int64_t*)malloc(sizeof(int64_t) * (size_t)(A->ptr[n] + 1));
  double* val = (double*)malloc(sizeof(double) * (size_t)(A->ptr[n] + 1));
  (void)nc;
  int64_t o = 0;
  ptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t b = o;
    double dii = 0.0;
    for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k) {
      if (A->col[k] == i) dii = A->val[k];
      const int64_t J = agg[A->col[k]];
      int64_t t = b;
      while (t < o && col[t] != J) ++t;
      if (t == o) { col[o] = J; val[o] = A->val[k]; ++o; }
      else val[t] = val[t] + A->val[k];
    }
    const double s = omega / dii;
    for (int64_t t = b; t < o; ++t) {
      const double v = s * val[t];
      val[t] = (col[t] == agg[i]) ? 1.0 - v : -v;
    }
    for (int64_t x = b + 1; x < o; ++x) { /* columns increasing */
      const int64_t cc = col[x];
      const double vv = val[x];
      int64_t y = x - 1;
      while (y >= b && col[y] > cc) { col[y + 1] = col[y]; val[y + 1] = val[y]; --y; }
      col[y + 1] = cc;
      val[y + 1] = vv;
    }
    ptr[i + 1] = o;
  }
  *pptr = ptr; *pcol = col; *pval = val;
}

/* R = P^T (explicit restriction, BASELINE.json north_star), rows by increasing column. */
void or_transpose(const or_csr* P, int64_t** rptr, int64_t** rcol, double** rval) {
  const int64_t n = P->nrows, nc = P->ncols, nnz = P->ptr[n];
  int64_t* ptr = (int64_t*)calloc((size_t)(nc + 1), sizeof(int64_t));
  int64_t* col = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz + 1));
  double* val = (double*)malloc(sizeof(double) * (size_t)(nnz + 1));
  for (int64_t k = 0; k < nnz; ++k) ptr[P->col[k] + 1]++;
  for (int64_t c = 0; c < nc; ++c) ptr[c + 1] += ptr[c];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nc + 1));
  memcpy(fill, ptr, sizeof(int64_t) * (size_t)(nc + 1));
  for (int64_t i = 0; i < n; ++i) /* rows of P in increasing i: each R row comes out sorted */
    for (int64_t k = P->ptr[i]; k < P->ptr[i + 1]; ++k) {
      const int64_t o = fill[P->col[k]]++;
      col[o] = i;
      val[o] = P->val[k];
    }
  free(fill);
  *rptr = ptr; *rcol = col; *rval = val;
}

/* Sparse product Z = X Y row by row (Gustavson):
 *   Z[i, K] = sum_{k in X_i} X_ik Y_kK
 * accumulated in that loop order (k, then K increasing), columns increasing; every
 * (i, K) reached is stored (also when the sum cancels). */
static void or_spgemm(const or_csr* X, const or_csr* Y, or_csr* Z) {
  const int64_t n = X->nrows, m = Y->ncols;
  double* acc = dalloc(m);
  int64_t* mark = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
  int64_t* touched = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
  for (int64_t K = 0; K < m; ++K) mark[K] = -1;
  int64_t cap = 1024, o = 0;
  int64_t* ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* col = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  double* val = (double*)malloc(sizeof(double) * (size_t)cap);
  ptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t nt = 0;
    for (int64_t b = X->ptr[i]; b < X->ptr[i + 1]; ++b) {
      const int64_t k = X->col[b];
      const double xv = X->val[b];
      for (int64_t c = Y->ptr[k]; c < Y->ptr[k + 1]; ++c) {
        const int64_t K = Y->col[c];
        if (mark[K] != i) { mark[K] = i; acc[K] = 0.0; touched[nt++] = K; }
        acc[K] = acc[K] + xv * Y->val[c];
      }
    }
    for (int64_t x = 1; x < nt; ++x) { /* sort the touched columns */
      const int64_t t = touched[x];
      int64_t y = x - 1;
      while (y >= 0 && touched[y] > t) { touched[y + 1] = touched[y]; --y; }
      touched[y + 1] = t;
    }
    if (o + nt > cap) {
      while (o + nt > cap) cap *= 2;
      col = (int64_t*)realloc(col, sizeof(int64_t) * (size_t)cap);
      val = (double*)realloc(val, sizeof(double) * (size_t)cap);
    }
    for (int64_t x = 0; x < nt; ++x) { col[o] = touched[x]; val[o] = acc[touched[x]]; ++o; }
    ptr[i + 1] = o;
  }
  free(acc); free(mark); free(touched);
  Z->nrows = n; Z->ncols = m; Z->ptr = ptr; Z->col = col; Z->val = val;
}

/* Galerkin coarse operator A_c = R A P (R = P^T), reading R31: associated
 * as R (A P), two sparse products in Gustavson's row order:
 *   (AP)[i, K] = sum_{k in A_i} a_ik P_kK,   A_c[J, K] = sum_{i in R_J} R_Ji (AP)[i, K]
 * (work nnz(A) * |P row| + nnz(R) * |AP row| instead of the triple product's
 * nnz(R) * |A row| * |P row|).  Same pattern as the triple product: every (J, K)
 * reached is stored. */
void or_galerkin(const or_csr* R, const or_csr* A, const or_csr* P, int64_t** cptr, int64_t** ccol,
                 double** cval) {
  or_csr AP, C;
  or_spgemm(A, P, &AP);
  or_spgemm(R, &AP, &C);
  free((void*)AP.ptr); free((void*)AP.col); free((void*)AP.val);
  *cptr = (int64_t*)C.ptr; *ccol = (int64_t*)C.col; *cval = (double*)C.val;
}

/* ======================================================================
 * NEXT-4: the AINV smoother (Sec. 2.3.2): "an approximate inverse of A
 * ... an incomplete biconjugation, approximating A_l^-1 as a product of two sparse
 * triangular matrices Z and W ... on GPUs ... only sparse matrix-vector products
 * with Z and W".  Reading R27: A symmetric positive definite, so W = Z and
 * A^-1 ~ Z D^-1 Z^T; right-looking biconjugation (Benzi-Meyer-Tuma):
 *   z_j = e_j (j = 0..n-1)
 *   for i = 0..n-1:  p_i = a_i^T z_i
 *       for j = i+1..n-1:  p_j = a_i^T z_j;  if p_j != 0: z_j = z_j - (p_j / p_i) z_i,
 *                          then drop the entries of z_j with |z_kj| < drop_tol (k != j)
 *   D = diag(p)
 * (a_i = row i of A; a_i^T z = sum over row i's entries in column order).  In the
 * distributed setting the paper's AINV inverts diagonal blocks (block-Jacobi): only
 * the columns of row_start's block of i are used.  The smoother M^-1 = Z D^-1 Z^T
 * replaces the l1-Jacobi M^-1 in Eq. (2).  Returns 0, or -1 - i if pivot p_i <= 0.
 * Z is returned by columns (zptr[n+1], zrow (increasing), zval) and p[n]. */
int or_ainv(const or_csr* A, int nranks, const int64_t* row_start, double drop_tol, int64_t** zptr,
            int64_t** zrow, double** zval, double* p) {
  const int64_t n = A->nrows;
  /* dense columns are the plain form of "z_j" for the small matrices the oracle sees */
  double* Z = (double*)calloc((size_t)(n * n > 0 ? n * n : 1), sizeof(double)); /* Z[k*n + j] = z_kj */
  int64_t* blk = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  for (int r = 0; r < nranks; ++r)
    for (int64_t i = row_start[r]; i < row_start[r + 1]; ++i) blk[i] = r;
  for (int64_t j = 0; j < n; ++j) Z[j * n + j] = 1.0;
  int status = 0;
  for (int64_t i = 0; i < n && status == 0; ++i) {
    double pi = 0.0;
    for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k)
      if (blk[A->col[k]] == blk[i]) pi += A->val[k] * Z[A->col[k] * n + i];
    p[i] = pi;
    if (!(pi > 0.0)) { status = (int)(-1 - i); break; }
    for (int64_t j = i + 1; j < n; ++j) {
      if (blk[j] != blk[i]) continue;
      double pj = 0.0;
      for (int64_t k = A->ptr[i]; k < A->ptr[i + 1]; ++k)
        if (blk[A->col[k]] == blk[i]) pj += A->val[k] * Z[A->col[k] * n + j];
      if (pj == 0.0) continue;
      const double f = pj / pi;
      for (int64_t k = 0; k <= i; ++k)
        if (Z[k * n + i] != 0.0) {
          Z[k * n + j] = Z[k * n + j] - f * Z[k * n + i];
          if (k != j && fabs(Z[k * n + j]) < drop_tol) Z[k * n + j] = 0.0;
        }
    }
  }
  int64_t nz = 0;
  for (int64_t q = 0; q < n * n; ++q) nz += Z[q] != 0.0;
  int64_t* cp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* rr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nz + 1));
  double* vv = (double*)malloc(sizeof(double) * (size_t)(nz + 1));
  int64_t o = 0;
  cp[0] = 0;
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t k = 0; k < n; ++k)
      if (Z[k * n + j] != 0.0) { rr[o] = k; vv[o] = Z[k * n + j]; ++o; }
    cp[j + 1] = o;
  }
  free(Z); free(blk);
  *zptr = cp; *zrow = rr; *zval = vv;
  return status;
}
