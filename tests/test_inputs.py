"""Checks of the seeded input generator (pscgen/): the given hierarchy must be
what PAPER.md Sec. 2.3 describes, independently of the oracle and the CUDA path.
All checks use scipy/numpy (library routines), closed forms and paper values."""
import numpy as np
import pytest
import scipy.sparse as sp

import pscgen
from _util import golden, grid_coords, poisson_eigpair, random_spd


@pytest.mark.parametrize("procs", [(1, 1, 1), (2, 1, 1), (1, 2, 2), (2, 2, 2)])
def test_A0_is_7point_poisson(procs):
    nx, ny, nz = 8, 6, 4
    h = pscgen.poisson_hierarchy(nx, ny, nz, procs, max_levels=1)
    A = h.levels[0].A.to_scipy()
    n = nx * ny * nz
    assert A.shape == (n, n) and A.nnz == 7 * n - 2 * (ny * nz + nx * nz + nx * ny)
    for ijk in ((1, 1, 1), (2, 5, 3), (nx, ny, nz)):
        lam, v = poisson_eigpair(nx, ny, nz, procs, *ijk)
        np.testing.assert_allclose(A @ v, lam * v, atol=1e-13)
    # strictly increasing columns per row
    for i in range(n):
        c = A.indices[A.indptr[i]:A.indptr[i + 1]]
        assert np.all(np.diff(c) > 0)
    # row blocks = rank boxes
    rs = h.levels[0].row_start
    assert list(rs) == [r * n // np.prod(procs) for r in range(np.prod(procs) + 1)]


def test_partition_is_a_permutation_of_the_single_rank_matrix():
    nx = 8
    h1 = pscgen.poisson_hierarchy(nx, max_levels=1)
    h8 = pscgen.poisson_hierarchy(nx, procs=(2, 2, 2), max_levels=1)
    gx, gy, gz = grid_coords(nx, nx, nx, (2, 2, 2))
    perm = gx + nx * (gy + nx * gz)  # row of the 8-rank numbering -> lexicographic index
    A1 = h1.levels[0].A.to_scipy()
    A8 = h8.levels[0].A.to_scipy()
    assert abs(A1[perm][:, perm] - A8).max() == 0


@pytest.mark.parametrize("problem,procs", [("poisson", (1, 1, 1)), ("poisson", (2, 2, 1)), ("jump", (1, 1, 2))])
def test_galerkin_hierarchy(problem, procs):
    """R_l = P_l^T exactly; A_{l+1} = R_l A_l P_l; coarse A symmetric and SPD."""
    h = pscgen.poisson_hierarchy(12, 12, 12, procs, problem=problem, cube=3, coarse_target=20)
    assert h.nlevels >= 3
    for l in range(h.nlevels - 1):
        L, N = h.levels[l], h.levels[l + 1]
        A, P, R = L.A.to_scipy(), L.P.to_scipy(), L.R.to_scipy()
        assert N.n < L.n
        assert abs(R - P.T.tocsr()).max() == 0
        Ac = N.A.to_scipy()
        ref = (R @ A @ P).toarray()
        assert np.abs(Ac.toarray() - ref).max() <= 1e-12 * np.abs(ref).max()
        assert abs(Ac - Ac.T).max() <= 1e-13 * abs(Ac).max()
        if Ac.shape[0] <= 2000:
            assert np.linalg.eigvalsh(Ac.toarray()).min() > 0


@pytest.mark.parametrize("procs", [(1, 1, 1), (2, 1, 2)])
def test_smoothed_prolongator_definition(procs):
    """P = (I - omega D^-1 A) P^ with omega = 1/||D^-1 A||_inf and the
    tentative P^ of Eq. (3) with w = 1; aggregates decoupled."""
    args = dict(nx=10, ny=10, nz=10, procs=procs, max_levels=2)
    hs = pscgen.poisson_hierarchy(args["nx"], args["ny"], args["nz"], procs, max_levels=2)
    ht = pscgen.poisson_hierarchy(args["nx"], args["ny"], args["nz"], procs, max_levels=2, smooth=False)
    A = hs.levels[0].A.to_scipy()
    Phat = ht.levels[0].P.to_scipy()
    # Eq. (3): exactly one entry w_i = 1 per row
    assert np.all(np.diff(Phat.indptr) == 1) and np.all(Phat.data == 1.0)
    # decoupled: fine row on rank r maps to a coarse column owned by rank r
    rs0, rs1 = hs.levels[0].row_start, hs.levels[1].row_start
    rank_f = np.searchsorted(rs0, np.arange(A.shape[0]), side="right") - 1
    rank_c = np.searchsorted(rs1, Phat.indices, side="right") - 1
    assert np.array_equal(rank_f, rank_c)
    Dinv = sp.diags(1.0 / A.diagonal())
    omega = 1.0 / abs(Dinv @ A).sum(axis=1).max()
    assert omega == pytest.approx(0.5, rel=1e-15)  # (6 + 6)/6 = 2 on the 7-point operator
    Pref = (sp.eye(A.shape[0]) - omega * Dinv @ A) @ Phat
    Ps = hs.levels[0].P.to_scipy()
    assert abs(Ps - Pref).max() <= 1e-15


def test_inf_norm_example_and_galerkin_example():
    # ||D^-1 A||_inf of tridiag n=2 = 1.5 -> omega = 2/3; S:303-294 Galerkin [[2,-1],[-1,2]], P=[1;1] -> [2]
    from _util import tridiag
    A = tridiag(2)
    P = sp.csr_matrix(np.ones((2, 1)))
    assert (P.T @ A @ P).toarray().tolist() == golden("galerkin_2x2_p_ones")
    assert abs(sp.diags(1 / A.diagonal()) @ A).sum(axis=1).max() == golden("inf_norm_Dinv_A_tridiag_n2")


def test_vmb_aggregates_are_strongly_connected_and_cover():
    """Every aggregate is a set of fine nodes; every node is aggregated (P^ has one
    entry per row) and every aggregate is non-empty (P^ has no empty column)."""
    h = pscgen.poisson_hierarchy(16, max_levels=2, smooth=False)
    Phat = h.levels[0].P.to_scipy().tocsc()
    assert np.all(np.diff(Phat.indptr) >= 1)
    assert Phat.shape[1] == h.levels[1].n


def test_operator_complexity_matches_paper():
    """Fig. 3: VBM operator complexity 1.575-1.59."""
    h = pscgen.poisson_hierarchy(64)
    lo, hi = golden("vbm_operator_complexity_range_all_gpus")
    assert lo - 0.02 <= h.operator_complexity() <= hi + 0.03


def test_jump_problem_reduces_to_poisson_at_unit_jump():
    hp = pscgen.poisson_hierarchy(8, max_levels=1)
    hj = pscgen.poisson_hierarchy(8, max_levels=1, problem="jump", jump=1.0, cube=2)
    assert abs(hp.levels[0].A.to_scipy() - hj.levels[0].A.to_scipy()).max() == 0
    hj = pscgen.poisson_hierarchy(8, max_levels=1, problem="jump", jump=1e4, cube=2)
    A = hj.levels[0].A.to_scipy()
    assert abs(A - A.T).max() == 0
    # weakly diagonally dominant M-matrix with at least one strictly dominant row
    off = np.asarray(abs(A).sum(axis=1)).ravel() - A.diagonal()
    assert np.all(A.diagonal() >= off) and np.any(A.diagonal() > off)


def test_rhs_random_keyed_by_global_index():
    full = pscgen.rhs_random(3, 0, 1000)
    assert np.array_equal(np.concatenate([pscgen.rhs_random(3, 0, 400), pscgen.rhs_random(3, 400, 600)]), full)
    assert full.min() >= -1.0 and full.max() < 1.0 and abs(full.mean()) < 0.1
    assert not np.array_equal(full, pscgen.rhs_random(4, 0, 1000))


def test_csr_hierarchy_general_matrix():
    A = random_spd(300, 0.02, 5)
    h = pscgen.csr_hierarchy(A, np.array([0, 150, 300]), coarse_target=10)
    assert h.nlevels >= 2
    for l in range(h.nlevels - 1):
        assert abs(h.levels[l].R.to_scipy() - h.levels[l].P.to_scipy().T).max() == 0


def test_csr_arrays_outlive_the_hierarchy_object():
    """The CSR arrays are views of C memory: they must keep the C hierarchy alive
    (a temporary hierarchy's matrix once read freed memory)."""
    import gc
    A = pscgen.poisson_hierarchy(6, max_levels=2).levels[0].A
    S = pscgen.poisson_hierarchy(5, max_levels=1).levels[0].A.to_scipy()
    gc.collect()
    junk = [np.ones(1 << 16) for _ in range(64)]  # reuse freed memory if it were freed
    assert A.ptr[0] == 0 and A.nnz == 6 ** 3 * 7 - 6 * 6 * 6
    assert S.indptr[0] == 0 and S.shape == (125, 125) and S.nnz == 725
    np.testing.assert_array_equal(S.diagonal(), np.full(125, 6.0))
    del junk


# ------------------------------------------ matching-based hierarchies (NEXT-3 set-up)
def test_matching_spec_examples():
    """SPEC S:263-278 (approx_max_weight_matching, matching_aggregate) with w = 1 and unit
    diagonals, so c_ij = 1 - a_ij (weights set through the couplings)."""
    import scipy.sparse as sp
    from _util import tridiag
    # path a-b-c with weights 1.2 then 1.5 -> (b, c) matched, a unmatched
    A = sp.csr_matrix(np.array([[1.0, -0.2, 0.0], [-0.2, 1.0, -0.5], [0.0, -0.5, 1.0]]))
    agg, ph, nc = pscgen.match(A, k=1)
    assert nc == 2 and agg[1] == agg[2] and agg[0] != agg[1]
    # triangle with equal weights -> exactly one edge (the lexicographically smallest), one vertex free
    T = sp.csr_matrix(np.array([[1.0, -0.3, -0.3], [-0.3, 1.0, -0.3], [-0.3, -0.3, 1.0]]))
    agg, ph, nc = pscgen.match(T, k=1)
    assert nc == 2 and agg[0] == agg[1] and agg[2] != agg[0]
    # 4-node path, uniform weights: k = 1 -> 2 pairs; k = 2 -> one aggregate of 4
    agg, ph, nc = pscgen.match(tridiag(4), k=1)
    assert nc == 2 and np.array_equal(agg, [0, 0, 1, 1])
    np.testing.assert_allclose(ph, np.full(4, 1 / np.sqrt(2)), rtol=1e-15)  # Eq. (4): (1,1)/sqrt(2)
    agg, ph, nc = pscgen.match(tridiag(4), k=2)
    assert nc == 1 and np.array_equal(agg, [0, 0, 0, 0])
    np.testing.assert_allclose(ph, np.full(4, 0.5), rtol=1e-15)
    # isolated vertex with w_s = 2 -> singleton, column entry 2/|2| = 1 (Eq. (4) W)
    agg, ph, nc = pscgen.match(sp.csr_matrix(np.array([[3.0]])), w=np.array([2.0]), k=1)
    assert nc == 1 and ph[0] == 1.0


def _brute_max_matching(n, edges):
    """Exact maximum weight matching by exhaustive recursion on the lowest free vertex."""
    wt = {}
    for c, i, j in edges:
        wt[(i, j)] = wt[(j, i)] = c

    def best(free):
        if not free:
            return 0.0
        v, rest = free[0], free[1:]
        b = best(rest)  # v unmatched
        for u in rest:
            if (v, u) in wt:
                b = max(b, wt[(v, u)] + best(tuple(x for x in rest if x != u)))
        return b

    return best(tuple(range(n)))


@pytest.mark.parametrize("seed", range(4))
def test_matching_half_approximation_and_orthonormal_prolongator(seed):
    """The greedy matching is a valid matching with weight >= 1/2 of the optimum (brute
    force on small graphs); P^ of Eq. (4) has orthonormal columns and w in its range."""
    import scipy.sparse as sp
    from _util import random_spd_mixed
    A = random_spd_mixed(9, 0.25, seed)
    w = 1.0 + np.random.default_rng(seed).random(9)
    agg, ph, nc = pscgen.match(A, w=w, k=1)
    Ad = A.toarray()
    d = np.diag(Ad)
    edges = []
    for i in range(9):
        for j in range(i + 1, 9):
            if Ad[i, j] != 0.0:
                c = 1.0 - 2.0 * Ad[i, j] * w[i] * w[j] / (d[i] * w[i] ** 2 + d[j] * w[j] ** 2)
                if c > 0:
                    edges.append((c, i, j))
    pairs = [np.flatnonzero(agg == a) for a in range(nc)]
    assert all(len(p) <= 2 for p in pairs)
    got = 0.0
    for p in pairs:
        if len(p) == 2:
            c = [e[0] for e in edges if e[1] == p[0] and e[2] == p[1]]
            assert c, p  # matched along a usable edge
            got += c[0]
    assert got >= 0.5 * _brute_max_matching(9, edges) - 1e-12
    P = sp.csr_matrix((ph, (np.arange(9), agg)), shape=(9, nc)).toarray()
    np.testing.assert_allclose(P.T @ P, np.eye(nc), rtol=0, atol=1e-14)
    np.testing.assert_allclose(P @ (P.T @ w), w, rtol=1e-14)


def test_matching_hierarchies_vs_paper_fig2_fig3():
    """SMATCH / VMATCH: aggregates of at most 8 = 2^3 nodes, smoothed / un-
    smoothed prolongators.  Operator complexity near Fig. 3's 1 GPU values (SMATCH 1.894,
    VMATCH 1.142; loose: the paper's matrix is 200^3, ours 64^3) and the
    iteration order of Fig. 2 at 1 GPU (SMATCH 9 < VBM 18 < VMATCH 28, P:380, P:399, P:418;
    FCG + coarsest PCG(40) to 1e-6 as in the paper's configurations)."""
    import oracle
    g = 64
    hs = pscgen.poisson_hierarchy(g, aggregation="matching", smooth=True)
    hv = pscgen.poisson_hierarchy(g, aggregation="matching", smooth=False)
    hb = pscgen.poisson_hierarchy(g)
    assert abs(hs.operator_complexity() - 1.894) <= 0.1
    assert abs(hv.operator_complexity() - 1.142) <= 0.01
    for h in (hs, hv):
        for l in range(h.nlevels - 1):
            assert h.levels[l].n <= 8 * h.levels[l + 1].n
    b = pscgen.rhs_poisson((g,) * 3, 0, g ** 3)
    kw = dict(coarse_pcg=True, coarse_maxit=40, coarse_tol=1e-10)
    its = oracle.fcg(hs, b, tol=1e-6, **kw)[1]
    itv = oracle.fcg(hv, b, tol=1e-6, pre=2, post=2, variable_v=True, **kw)[1]
    itb = oracle.fcg(hb, b, tol=1e-6, **kw)[1]
    assert abs(its - 9) <= 3
    assert its < itb < itv
