"""Pins of the CPU oracle (oracle/psc_oracle.c) to things other than itself:
values printed in the paper / SPEC worked examples (tests/golden), closed forms,
invariants, library routines (dense numpy/scipy), brute force on tiny inputs.

Each oracle function is pinned so that a plausible mistake (dropped term, wrong
sign or index, transposed operand) fails at least one test here:

  or_spmv            -> S:79 example, dense matmul, Poisson closed-form eigenpairs
  or_l1_diag         -> S:374-375 literal values, corner/edge/face values of 7-point
  or_l1_sweep(s)     -> fixed point, closed form (I - G^k) A^-1 b, A-norm decrease,
                        rho(I - M^-1 A) < 1 ("A_l-convergent")
  or_vcycle          -> dense Eq. (2) composition on 2- and 3-level
                        hierarchies, symmetry, SPD, ||I - BA||_A < 1, linearity;
                        variable V-cycle (P:330 footnote) vs dense Eq. (2) with
                        G_l^(pre 2^l), 2-level special case, symmetry/SPD
  or_pcg             -> Cholesky / DST exact solve, scipy's CG with the same B,
                        A = I, diag(1..10), b = 0, A-norm error monotone,
                        true vs recurrence residual, paper Fig. 2 loose pin
  or_coarse_pcg      -> S:417-418 examples, scipy CG with M = diag(1/m) iterate by
                        iterate, exact-coarse V-cycle = dense Eq. (2) with A^-1
  or_fcg             -> PCG iterates for a fixed SPD B (Notay FCG(1)), Cholesky,
                        A = I, b = 0, variable-B convergence, VBM loose pin
"""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

import oracle
import pscgen
from _util import golden, poisson_eigpair, poisson_exact_solve, random_spd, random_spd_mixed, tridiag


# ------------------------------------------------------------------ or_spmv
def test_spmv_spec_examples():
    # S:78 A = I3 -> x ; S:79 tridiag(-1,2,-1) n=3 times ones -> (1,0,1)
    x = np.array([1.0, 2.0, 3.0])
    assert np.array_equal(oracle.spmv(sp.eye(3, format="csr"), x), x)
    assert np.array_equal(oracle.spmv(tridiag(3), np.ones(3)), np.array(golden("spmv_tridiag3_ones")))


def test_spmv_matches_dense_rectangular():
    rng = np.random.default_rng(0)
    for m, n in ((17, 40), (40, 17), (64, 64)):
        A = sp.random(m, n, density=0.2, random_state=rng, format="csr")
        x = rng.standard_normal(n)
        np.testing.assert_allclose(oracle.spmv(A, x), A.toarray() @ x, rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("dims,procs", [((5, 5, 5), (1, 1, 1)), ((6, 4, 8), (2, 2, 2)), ((8, 6, 4), (2, 1, 1))])
def test_spmv_poisson_closed_form_eigenpairs(dims, procs):
    """A v = lambda v for the unscaled 7-point operator (closed-form spectrum)."""
    nx, ny, nz = dims
    h = pscgen.poisson_hierarchy(nx, ny, nz, procs, max_levels=1)
    A = h.levels[0].A
    for (i, j, k) in ((1, 1, 1), (2, 3, 1), (nx, ny, nz), (3, 1, 2)):
        lam, v = poisson_eigpair(nx, ny, nz, procs, i, j, k)
        np.testing.assert_allclose(oracle.spmv(A, v), lam * v, rtol=0, atol=1e-13)


# --------------------------------------------------------------- or_l1_diag
def test_l1_diag_spec_values():
    assert np.array_equal(oracle.l1_diag(tridiag(4)), np.array(golden("l1_diag_tridiag_n4")))
    # diagonal A -> m = diag(A)
    d = np.array([1.0, 2.5, 7.0])
    assert np.array_equal(oracle.l1_diag(sp.diags(d, format="csr")), d)


def test_l1_diag_poisson_corner_edge_face_interior():
    """7-point (6,-1): m = 6 + #neighbours: interior 12, face 11, edge 10, corner 9."""
    h = pscgen.poisson_hierarchy(5, max_levels=1)
    m = oracle.l1_diag(h.levels[0].A)
    from _util import grid_coords
    gx, gy, gz = grid_coords(5, 5, 5, (1, 1, 1))
    nb = sum(((c > 0).astype(int) + (c < 4).astype(int)) for c in (gx, gy, gz))
    assert np.array_equal(m, 6.0 + nb)
    assert m[(gx == 2) & (gy == 2) & (gz == 2)][0] == golden("l1_diag_poisson7_interior")
    assert set(np.unique(m)) == {9.0, 10.0, 11.0, 12.0}


def test_l1_diag_uses_abs_of_offdiag_and_signed_diag():
    A = sp.csr_matrix(np.array([[4.0, 1.0, -2.0], [1.0, 3.0, 0.0], [-2.0, 0.0, 5.0]]))
    assert np.array_equal(oracle.l1_diag(A), np.array([7.0, 4.0, 7.0]))


# -------------------------------------------------------------- or_l1_sweep
def _M(A):
    A = sp.csr_matrix(A)
    d = A.diagonal()
    return d + (np.asarray(abs(A).sum(axis=1)).ravel() - np.abs(d))


def test_sweep_fixed_point_and_one_sweep_formula():
    A = random_spd(60, 0.08, 1)
    rng = np.random.default_rng(2)
    b = rng.standard_normal(60)
    xs = np.linalg.solve(A.toarray(), b)
    np.testing.assert_allclose(oracle.l1_sweep(A, b, xs), xs, rtol=0, atol=1e-12)
    x = rng.standard_normal(60)
    expect = x + (b - A.toarray() @ x) / _M(A)
    np.testing.assert_allclose(oracle.l1_sweep(A, b, x), expect, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_sweeps_from_zero_closed_form(seed):
    """k sweeps from x=0: x_k = (I - G^k) A^{-1} b with G = I - M^{-1} A."""
    A = random_spd_mixed(40, 0.05, seed)
    Ad = A.toarray()
    b = np.random.default_rng(seed).standard_normal(40)
    G = np.eye(40) - Ad / _M(A)[:, None]
    for k in (1, 2, 5, 30):
        xk = (np.eye(40) - np.linalg.matrix_power(G, k)) @ np.linalg.solve(Ad, b)
        np.testing.assert_allclose(oracle.l1_sweeps_from_zero(A, b, k), xk, rtol=1e-9, atol=1e-11)


@pytest.mark.parametrize("seed", range(5))
def test_l1_jacobi_is_A_convergent(seed):
    """l1-Jacobi "is A_l-convergent": rho(I - M^-1 A) < 1 and the A-norm
    of the error decreases every sweep."""
    A = random_spd_mixed(50, 0.06, 10 + seed)
    Ad = A.toarray()
    m = oracle.l1_diag(A)
    G = np.eye(50) - Ad / m[:, None]
    assert np.max(np.abs(np.linalg.eigvals(G))) < 1.0
    rng = np.random.default_rng(seed)
    b = rng.standard_normal(50)
    xs = np.linalg.solve(Ad, b)
    x = np.zeros(50)
    prev = np.inf
    for _ in range(10):
        x = oracle.l1_sweep(A, b, x)
        e = x - xs
        en = np.sqrt(e @ Ad @ e)
        assert en < prev
        prev = en


# ---------------------------------------------------------------- or_vcycle
def _dense_B(hier, pre, post, coarse, variable_v=False):
    """B_0 from the error-propagation form of Eq. (2), built with dense
    matrices, recursively; B_ell = (I - G^coarse) A^-1 at the coarsest level.
    variable_v: level l smooths pre*2^l / post*2^l times (P:330 footnote, R25)."""
    L = hier.nlevels

    def Bl(l):
        A = hier.levels[l].A.to_scipy().toarray()
        n = A.shape[0]
        G = np.eye(n) - A / _M(A)[:, None]
        if l == L - 1:
            return (np.eye(n) - np.linalg.matrix_power(G, coarse)) @ np.linalg.inv(A)
        P = hier.levels[l].P.to_scipy().toarray()
        R = hier.levels[l].R.to_scipy().toarray()
        k = 2 ** l if variable_v else 1
        E = (np.linalg.matrix_power(G, post * k) @ (np.eye(n) - P @ Bl(l + 1) @ R @ A)
             @ np.linalg.matrix_power(G, pre * k))
        return (np.eye(n) - E) @ np.linalg.inv(A)

    return Bl(0)


def _oracle_B(hier, pre, post, coarse, **kw):
    n = hier.levels[0].n
    return np.column_stack([oracle.vcycle(hier, e, pre, post, coarse, **kw) for e in np.eye(n)])


@pytest.mark.parametrize("grid,procs,maxl,opts", [
    (6, (1, 1, 1), 2, (4, 4, 30)),
    (6, (1, 1, 1), 3, (4, 4, 30)),
    (6, (2, 1, 1), 3, (2, 3, 7)),
    (8, (2, 2, 1), 3, (1, 1, 5)),
])
def test_vcycle_equals_dense_eq2(grid, procs, maxl, opts):
    h = pscgen.poisson_hierarchy(grid, grid, grid, procs, max_levels=maxl, coarse_target=1)
    assert h.nlevels == maxl
    Bo = _oracle_B(h, *opts)
    Bd = _dense_B(h, *opts)
    np.testing.assert_allclose(Bo, Bd, rtol=0, atol=1e-11 * np.abs(Bd).max())


@pytest.mark.parametrize("problem", ["poisson", "jump"])
def test_vcycle_symmetric_spd_contractive(problem):
    """Equal pre/post l1-Jacobi (diagonal M, M^-T = M^-1) gives a symmetric B (R9);
    B is SPD and ||I - BA||_A < 1 (multigrid convergence)."""
    h = pscgen.poisson_hierarchy(8, problem=problem, cube=2, coarse_target=10)
    assert h.nlevels >= 3
    B = _oracle_B(h, 4, 4, 30)
    assert np.linalg.norm(B - B.T) / np.linalg.norm(B) < 1e-13
    w = np.linalg.eigvalsh(0.5 * (B + B.T))
    assert w.min() > 0
    A = h.levels[0].A.to_scipy().toarray()
    Lc = np.linalg.cholesky(A)
    E = Lc.T @ (np.eye(A.shape[0]) - B @ A) @ np.linalg.inv(Lc.T)  # A-norm similarity
    assert np.linalg.norm(E, 2) < 1.0


def test_vcycle_unequal_sweeps_not_symmetric():
    """Sanity of the symmetry pin: pre != post breaks symmetry (so the test above can fail)."""
    h = pscgen.poisson_hierarchy(6, max_levels=2)
    B = _oracle_B(h, 1, 3, 30)
    assert np.linalg.norm(B - B.T) / np.linalg.norm(B) > 1e-6


@pytest.mark.parametrize("grid,procs,maxl,opts", [
    (6, (1, 1, 1), 3, (2, 2, 30)),
    (8, (2, 1, 1), 4, (1, 2, 7)),
])
def test_variable_vcycle_equals_dense_eq2(grid, procs, maxl, opts):
    """Variable V-cycle (P:330 footnote, R25): sweeps pre*2^l / post*2^l at level l,
    against the dense Eq. (2) composition with those powers of G_l."""
    h = pscgen.poisson_hierarchy(grid, grid, grid, procs, max_levels=maxl, coarse_target=1)
    assert h.nlevels == maxl
    Bo = _oracle_B(h, *opts, variable_v=True)
    Bd = _dense_B(h, *opts, variable_v=True)
    np.testing.assert_allclose(Bo, Bd, rtol=0, atol=1e-11 * np.abs(Bd).max())
    # and it is a different operator from the plain V-cycle (level 1 smooths twice as often)
    assert np.abs(Bo - _oracle_B(h, *opts)).max() > 1e-6 * np.abs(Bd).max()


def test_variable_vcycle_two_levels_is_plain_vcycle():
    """Special case: with two levels only level 0 smooths, and 2^0 = 1, so the variable
    V-cycle is the plain V-cycle bit for bit."""
    h = pscgen.poisson_hierarchy(6, max_levels=2)
    r = np.random.default_rng(3).standard_normal(h.levels[0].n)
    assert np.array_equal(oracle.vcycle(h, r, 2, 2, 30, variable_v=True), oracle.vcycle(h, r, 2, 2, 30))


def test_variable_vcycle_symmetric_spd():
    """Equal pre/post counts stay equal at every level under doubling, so B stays
    symmetric and SPD (PCG-admissible) and ||I - BA||_A < 1."""
    h = pscgen.poisson_hierarchy(8, problem="jump", cube=2, coarse_target=10)
    assert h.nlevels >= 3
    B = _oracle_B(h, 2, 2, 30, variable_v=True)
    assert np.linalg.norm(B - B.T) / np.linalg.norm(B) < 1e-13
    assert np.linalg.eigvalsh(0.5 * (B + B.T)).min() > 0
    A = h.levels[0].A.to_scipy().toarray()
    Lc = np.linalg.cholesky(A)
    E = Lc.T @ (np.eye(A.shape[0]) - B @ A) @ np.linalg.inv(Lc.T)
    assert np.linalg.norm(E, 2) < 1.0


def test_vcycle_linear():
    h = pscgen.poisson_hierarchy(16, coarse_target=50)
    rng = np.random.default_rng(3)
    u, v = rng.standard_normal((2, h.levels[0].n))
    assert np.array_equal(oracle.vcycle(h, np.zeros(h.levels[0].n)), np.zeros(h.levels[0].n))
    lhs = oracle.vcycle(h, 2.5 * u + v)
    rhs = 2.5 * oracle.vcycle(h, u) + oracle.vcycle(h, v)
    np.testing.assert_allclose(lhs, rhs, rtol=0, atol=1e-12 * np.abs(rhs).max())


# -------------------------------------------------------------------- or_pcg
def test_pcg_matches_cholesky_tiny():
    h = pscgen.poisson_hierarchy(6, coarse_target=20)
    A = h.levels[0].A.to_scipy().toarray()
    b = pscgen.rhs_random(7, 0, h.levels[0].n)
    x, it, st, hist = oracle.pcg(h, b, tol=1e-13, maxit=216)
    assert st == 0 and it <= 216
    xc = sla.cho_solve(sla.cho_factor(A), b)
    assert np.linalg.norm(x - xc) / np.linalg.norm(xc) < 1e-11


@pytest.mark.parametrize("n", [8, 16])
def test_pcg_matches_dst_exact_poisson(n):
    h = pscgen.poisson_hierarchy(n, procs=(2, 1, 1))
    b = pscgen.rhs_poisson((n, n, n), 0, h.levels[0].n)
    x, it, st, hist = oracle.pcg(h, b, tol=1e-11, maxit=100)
    assert st == 0
    xs = poisson_exact_solve(n, n, n, (2, 1, 1), b)
    assert np.linalg.norm(x - xs) / np.linalg.norm(xs) < 1e-9
    # true residual agrees with the recurrence residual at exit
    A = h.levels[0].A.to_scipy()
    true = np.linalg.norm(b - A @ x) / np.linalg.norm(b)
    assert abs(true - hist[-1]) <= 1e-12 + 0.01 * hist[-1]


def test_pcg_identity_diag_and_zero_rhs():
    # S:470 A = I -> 1 iteration
    hI = pscgen.csr_hierarchy(sp.eye(20, format="csr"))
    b = np.arange(1.0, 21.0)
    x, it, st, _ = oracle.pcg(hI, b, tol=1e-12)
    assert st == 0 and it == 1 and np.allclose(x, b, rtol=1e-15)
    # S:471 diag(1..10) -> <= 10 iterations
    hD = pscgen.csr_hierarchy(sp.diags(np.arange(1.0, 11.0), format="csr"))
    x, it, st, _ = oracle.pcg(hD, np.ones(10), tol=1e-12)
    assert st == 0 and it <= 10
    np.testing.assert_allclose(x, 1.0 / np.arange(1.0, 11.0), rtol=1e-11)
    # S:472 b = 0 -> 0 iterations, x = 0
    h = pscgen.poisson_hierarchy(6, max_levels=2)
    x, it, st, hist = oracle.pcg(h, np.zeros(216), x0=np.ones(216))
    assert st == 0 and it == 0 and not x.any()


def test_pcg_iterates_equal_scipy_cg_with_same_preconditioner():
    """The PCG recurrence against scipy.sparse.linalg.cg (independent Krylov code)
    using the oracle's V-cycle as M: iterates x_k agree for every k."""
    from scipy.sparse.linalg import LinearOperator, cg
    h = pscgen.poisson_hierarchy(12, coarse_target=30)
    n = h.levels[0].n
    A = h.levels[0].A.to_scipy()
    b = pscgen.rhs_random(11, 0, n)
    M = LinearOperator((n, n), matvec=lambda r: oracle.vcycle(h, np.asarray(r).ravel()))
    for k in (1, 2, 4, 6):
        xo, it, st, _ = oracle.pcg(h, b, tol=0.0, maxit=k)
        assert it == k and st == 1
        xs, info = cg(A, b, x0=np.zeros(n), rtol=0.0, atol=0.0, maxiter=k, M=M)
        np.testing.assert_allclose(xo, xs, rtol=0, atol=1e-10 * np.abs(xs).max())


def test_pcg_A_norm_error_monotone():
    h = pscgen.poisson_hierarchy(10, procs=(1, 2, 1), coarse_target=30)
    n = h.levels[0].n
    A = h.levels[0].A.to_scipy()
    b = pscgen.rhs_random(5, 0, n)
    xs = sla.cho_solve(sla.cho_factor(A.toarray()), b)
    prev = np.inf
    for k in range(1, 9):
        x, it, st, _ = oracle.pcg(h, b, tol=0.0, maxit=k)
        e = x - xs
        en = np.sqrt(e @ (A @ e))
        assert en < prev
        prev = en


def test_pcg_breakdown_on_indefinite():
    # An indefinite symmetric matrix with a hierarchy of one level: p^T A p <= 0 -> status -6.
    A = sp.csr_matrix(np.array([[1.0, 0.0], [0.0, -1.0]]))
    h = pscgen.csr_hierarchy(A, max_levels=1)
    x, it, st, _ = oracle.pcg(h, np.array([1.0, 1.0]), tol=1e-12, pre=1, post=1, coarse=1)
    assert st == -6


@pytest.mark.slow
def test_paper_fig2_iterations_loose():
    """PAPER.md Fig. 2: VBM needs 18 iterations at 1 GPU to tol 1e-6 on
    8e6 dof.  Our configuration differs (PCG vs FCG, 30 coarse sweeps vs PCG(40),
    128^3 vs 200^3), so this is a loose pin: within +-4 iterations."""
    h = pscgen.poisson_hierarchy(128)
    b = pscgen.rhs_poisson((128, 128, 128), 0, h.levels[0].n)
    x, it, st, hist = oracle.pcg(h, b, tol=1e-6, maxit=100)
    assert st == 0
    assert abs(it - golden("vbm_iterations_1gpu_tol1e-6")) <= 4


# ------------------------------------------- NEXT-2: coarse PCG(40) and FCG(1)
def test_coarse_pcg_spec_examples():
    # [2] x = 4 -> x = 2 ; diag(1..5) exact within 5 iterations
    x, it = oracle.coarse_pcg(sp.csr_matrix(np.array([[2.0]])), np.array([4.0]), maxit=40, tol=1e-12)
    assert it == 1 and x[0] == 2.0
    x, it = oracle.coarse_pcg(sp.diags(np.arange(1.0, 6.0), format="csr"), np.ones(5), maxit=40, tol=1e-12)
    assert it <= 5
    np.testing.assert_allclose(x, 1.0 / np.arange(1.0, 6.0), rtol=1e-14)


@pytest.mark.parametrize("seed", [0, 1])
def test_coarse_pcg_iterates_equal_scipy_cg(seed):
    """P:328 "PCG coupled to l1-Jacobi preconditioner": iterates equal scipy's CG with
    M^{-1} = diag(1/m), m = a_ii + sum_{j!=i} |a_ij| (S:374 values pinned above)."""
    from scipy.sparse.linalg import LinearOperator, cg
    A = random_spd_mixed(40, 0.08, seed)
    b = np.random.default_rng(seed).standard_normal(40)
    m = oracle.l1_diag(A)
    M = LinearOperator((40, 40), matvec=lambda r: np.asarray(r).ravel() / m)
    for k in (1, 2, 5, 9):
        xo, it = oracle.coarse_pcg(A, b, maxit=k, tol=0.0)
        assert it == k
        xs, _ = cg(A, b, x0=np.zeros(40), rtol=0.0, atol=0.0, maxiter=k, M=M)
        np.testing.assert_allclose(xo, xs, rtol=0, atol=1e-11 * np.abs(xs).max())
    xo, it = oracle.coarse_pcg(A, b, maxit=400, tol=1e-13)
    np.testing.assert_allclose(xo, np.linalg.solve(A.toarray(), b), rtol=1e-10, atol=1e-12)


def test_vcycle_with_exact_coarse_pcg_equals_dense_eq2():
    """Coarse PCG run to exactness (maxit >= n_coarse, tiny tol) is B_ell = A_ell^{-1} in Eq. (2)."""
    h = pscgen.poisson_hierarchy(6, max_levels=3, coarse_target=1)
    n = h.levels[0].n
    L = h.nlevels
    # dense Eq. (2) with an exact coarsest solve
    def Bl(l):
        A = h.levels[l].A.to_scipy().toarray()
        if l == L - 1:
            return np.linalg.inv(A)
        G = np.eye(A.shape[0]) - A / _M(A)[:, None]
        P = h.levels[l].P.to_scipy().toarray()
        R = h.levels[l].R.to_scipy().toarray()
        E = np.linalg.matrix_power(G, 4) @ (np.eye(A.shape[0]) - P @ Bl(l + 1) @ R @ A) @ np.linalg.matrix_power(G, 4)
        return (np.eye(A.shape[0]) - E) @ np.linalg.inv(A)
    Bd = Bl(0)
    r = pscgen.rhs_random(3, 0, n)
    z = oracle.vcycle(h, r, coarse_pcg=True, coarse_maxit=1000, coarse_tol=1e-15)
    np.testing.assert_allclose(z, Bd @ r, rtol=0, atol=1e-10 * np.abs(Bd @ r).max())


def test_fcg_equals_pcg_for_fixed_spd_preconditioner():
    """Notay's FCG(1) and PCG build the same iterates for a fixed SPD B (exact arithmetic;
    S:476): compare x_k for every k with the pinned PCG."""
    h = pscgen.poisson_hierarchy(12, coarse_target=30)
    b = pscgen.rhs_random(21, 0, h.levels[0].n)
    for k in (1, 2, 3, 5, 8):
        xp, ip, sp_, _ = oracle.pcg(h, b, tol=0.0, maxit=k)
        xf, if_, sf, _ = oracle.fcg(h, b, tol=0.0, maxit=k)
        assert ip == if_ == k
        np.testing.assert_allclose(xf, xp, rtol=0, atol=1e-10 * np.abs(xp).max())


def test_fcg_cholesky_identity_zero_rhs():
    h = pscgen.poisson_hierarchy(6, coarse_target=20)
    A = h.levels[0].A.to_scipy().toarray()
    b = pscgen.rhs_random(8, 0, h.levels[0].n)
    x, it, st, hist = oracle.fcg(h, b, tol=1e-13, maxit=216)
    assert st == 0
    xc = sla.cho_solve(sla.cho_factor(A), b)
    assert np.linalg.norm(x - xc) / np.linalg.norm(xc) < 1e-11
    hI = pscgen.csr_hierarchy(sp.eye(20, format="csr"))
    x, it, st, _ = oracle.fcg(hI, np.arange(1.0, 21.0), tol=1e-12)
    assert st == 0 and it == 1
    x, it, st, _ = oracle.fcg(h, np.zeros(h.levels[0].n), x0=np.ones(h.levels[0].n))
    assert st == 0 and it == 0 and not x.any()


def test_fcg_with_variable_coarse_pcg_converges():
    """A loose coarse PCG (tol 1e-2) makes B vary between applications: FCG still
    converges and its recurrence residual matches the true residual."""
    h = pscgen.poisson_hierarchy(16, coarse_target=60)
    b = pscgen.rhs_poisson((16, 16, 16), 0, h.levels[0].n)
    x, it, st, hist = oracle.fcg(h, b, tol=1e-10, maxit=100, coarse_pcg=True, coarse_maxit=40, coarse_tol=1e-2)
    assert st == 0
    A = h.levels[0].A.to_scipy()
    true = np.linalg.norm(b - A @ x) / np.linalg.norm(b)
    assert true <= 1e-9


@pytest.mark.slow
def test_paper_vbm_configuration_iterations_loose():
    """The paper's VBM solve: FCG, l1-Jacobi V-cycle, coarsest PCG(<= 40)
    with l1-Jacobi; Fig. 2: 18 iterations to 1e-6 on 8e6 dof (loose +-4 at 128^3)."""
    h = pscgen.poisson_hierarchy(128)
    b = pscgen.rhs_poisson((128, 128, 128), 0, h.levels[0].n)
    x, it, st, hist = oracle.fcg(h, b, tol=1e-6, maxit=100, coarse_pcg=True, coarse_maxit=40, coarse_tol=1e-10)
    assert st == 0
    assert abs(it - golden("vbm_iterations_1gpu_tol1e-6")) <= 4


# ----------------------- FCG(1)'s flexible update and the coarse PCG's stop rule
# (VERDICT r1 "What's weak" 1: a Fletcher-Reeves mutant of or_fcg passed every pin
# above, because all of them use a fixed -- or nearly fixed -- preconditioner.)
_VARB = dict(coarse_pcg=True, coarse_maxit=2, coarse_tol=0.0)  # B(r) strongly nonlinear in r


def _iterates(solve, h, b, K, **kw):
    """x_0 .. x_K of a Krylov solve (each x_k from a fresh run with maxit = k; the runs
    are deterministic, so x_k of the run with maxit = K is the same vector)."""
    xs = [np.zeros_like(b)]
    for k in range(1, K + 1):
        x, it, st, _ = solve(h, b, tol=0.0, maxit=k, **kw)
        assert it == k
        xs.append(x)
    return xs


def test_fcg_local_a_orthogonality_with_variable_preconditioner():
    """Notay's FCG(1) (reading R24) A-orthogonalises each new direction
    against the previous one, p_k = z_k - ((z_k, A p_{k-1})/(p_{k-1}, A p_{k-1})) p_{k-1},
    so (p_k, A p_{k-1}) = 0 for ANY z_k -- also when B varies between applications.
    The directions are recovered from the iterates, p_k ∝ x_k - x_{k-1}.  Exact line
    search alpha_k = (p_k, r_{k-1})/(p_k, A p_k) makes r_k ⟂ p_k.  PCG's Fletcher-Reeves
    beta = (r,z)_k/(r,z)_{k-1} gives neither property once B is nonlinear (the coarse
    PCG with 2 iterations and no tolerance), which the last assertion checks so
    that the regime is known to discriminate."""
    h = pscgen.poisson_hierarchy(16, max_levels=2)
    assert h.levels[-1].n > 500
    A = h.levels[0].A.to_scipy()
    b = pscgen.rhs_random(17, 0, h.levels[0].n)
    K = 7

    def worst_orth(xs):
        d = [xs[k] - xs[k - 1] for k in range(1, K + 1)]
        an = [np.sqrt(v @ (A @ v)) for v in d]
        return max(abs(d[k] @ (A @ d[k - 1])) / (an[k] * an[k - 1]) for k in range(1, K))

    xf = _iterates(oracle.fcg, h, b, K, **_VARB)
    assert worst_orth(xf) <= 1e-12
    for k in range(1, K + 1):
        d, r = xf[k] - xf[k - 1], b - A @ xf[k]
        assert abs(d @ r) <= 1e-12 * np.linalg.norm(d) * np.linalg.norm(b)
    xp = _iterates(oracle.pcg, h, b, K, **_VARB)
    assert worst_orth(xp) >= 1e-4  # PCG loses local A-orthogonality with this B


def test_fcg_differs_from_pcg_with_variable_preconditioner():
    """With a strongly nonlinear B the flexible and the Fletcher-Reeves recurrences build
    different iterates (they coincide only for a fixed SPD B, pinned above); FCG
    still converges, with the recurrence residual equal to the true one."""
    h = pscgen.poisson_hierarchy(16, max_levels=2)
    A = h.levels[0].A.to_scipy()
    b = pscgen.rhs_random(18, 0, h.levels[0].n)
    _, itf, stf, hf = oracle.fcg(h, b, tol=1e-10, maxit=200, **_VARB)
    _, itp, stp, hp = oracle.pcg(h, b, tol=1e-10, maxit=200, **_VARB)
    k = min(itf, itp, 10) + 1
    assert np.max(np.abs(hf[2:k] - hp[2:k]) / hp[2:k]) > 1e-6
    x, it, st, hist = oracle.fcg(h, b, tol=1e-10, maxit=200, **_VARB)
    assert st == 0
    assert np.linalg.norm(b - A @ x) / np.linalg.norm(b) <= 1e-9


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("tol", [1e-2, 1e-4, 1e-6])
def test_coarse_pcg_stop_rule_equals_first_k_below_tol(seed, tol):
    """Reading R23 (P:328 gives no test): stop at the first k with ||r_k||_2 <= tol ||b||_2
    (x_0 = 0).  Pinned against scipy's CG with M^{-1} = diag(1/m) run without its own
    test: the oracle's count is the first k whose scipy iterate has a true residual below
    tol ||b||, and the oracle's x is that iterate.  A squared norm, a ||r_0|| or ||z||
    denominator, or an off-by-one in the count fails this."""
    from scipy.sparse.linalg import LinearOperator, cg
    n = 80
    A = random_spd(n, 0.08, 3 + seed)
    b = np.random.default_rng(seed).standard_normal(n) * 7.0
    m = oracle.l1_diag(A)
    M = LinearOperator((n, n), matvec=lambda r: np.asarray(r).ravel() / m)
    xs = []
    cg(A, b, x0=np.zeros(n), rtol=0.0, atol=0.0, maxiter=300, M=M, callback=lambda xk: xs.append(xk.copy()))
    res = [np.linalg.norm(b - A @ x) / np.linalg.norm(b) for x in xs]
    kstar = next(k for k, r in enumerate(res, start=1) if r <= tol)
    assert res[kstar - 1] < (1 - 1e-6) * tol and (kstar == 1 or res[kstar - 2] > (1 + 1e-6) * tol)  # no rounding tie
    xo, it = oracle.coarse_pcg(A, b, maxit=300, tol=tol)
    assert it == kstar
    np.testing.assert_allclose(xo, xs[kstar - 1], rtol=0, atol=1e-10 * np.abs(xs[kstar - 1]).max())
    xo, it = oracle.coarse_pcg(A, b, maxit=kstar - 1, tol=tol)  # the cap wins when it comes first
    assert it == kstar - 1


# ------------------------------------------------------ OpenMP build of the oracle
def test_openmp_oracle_build_is_bitwise_identical():
    """SURVEY.md §8(d) "Oracle timing": the OpenMP build (cpu_baseline on all host cores)
    computes exactly what the serial build does (row-parallel loops, fixed-chunk dots)."""
    import os
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path[:0] = [%r, %r]\n"
        "import oracle, pscgen\n"
        "t = oracle.set_threads(int(sys.argv[1]))\n"
        "h = pscgen.poisson_hierarchy(24, 20, 16, coarse_target=40)\n"
        "b = pscgen.rhs_random(5, 0, h.levels[0].n)\n"
        "x, it, st, hist = oracle.pcg(h, b, tol=1e-10)\n"
        "xf, itf, stf, hf = oracle.fcg(h, b, tol=1e-10, coarse_pcg=True, coarse_maxit=7, coarse_tol=1e-3)\n"
        "np.save(sys.argv[2], np.concatenate([x, hist, xf, hf, [it, itf, t]]))\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__)))
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        outs = []
        for nt in (1, 4):
            f = os.path.join(d, f"o{nt}.npy")
            subprocess.check_call([sys.executable, "-c", code, str(nt), f])
            outs.append(np.load(f))
    assert outs[1][-1] == 4 and outs[0][-1] == 1
    assert np.array_equal(outs[0][:-1], outs[1][:-1])
