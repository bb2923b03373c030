"""Pins of the oracle's set-up (oracle/psc_oracle.c
or_vmb_aggregate, or_omega, or_smoothed_prolongator, or_transpose, or_galerkin):
decoupled VMB aggregation, the tentative prolongator of Eq. (3) with
w = 1, its smoothing with omega = 1/||D^-1 A||_inf, R = P^T,
and the Galerkin product A_{l+1} = P^T A P.  Readings R17-R21, R26.

Pinned against: SPEC.md worked examples, the
characterisation of a greedy distance-2 independent set (independence + every
non-root has a smaller-index root within two strong edges -- which determines the
set uniquely), the phase-1 / phase-2 rules checked node by node from the strength
definition, closed forms (omega = 1/2 on 7-point Poisson, P 1 = (I - omega D^-1 A) 1,
omega = 0 gives P^ of Eq. (3)), the bilinear identity of the Galerkin product,
symmetry / SPD, and the paper's operator complexity (Fig. 3) and
iteration count (Fig. 2) loosely.
"""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import shortest_path

import oracle
import pscgen
from _util import golden, random_spd_mixed, tridiag


def _strong(A, theta, row_start):
    """N_i(theta) of P:215-216 restricted to the row block of i (decoupled, R20):
    boolean sparse matrix S, S_ij = 1 iff j != i and |a_ij| >= theta sqrt(a_ii a_jj)."""
    A = sp.csr_matrix(A)
    n = A.shape[0]
    blk = np.zeros(n, np.int64)
    for r in range(len(row_start) - 1):
        blk[row_start[r]:row_start[r + 1]] = r
    d = A.diagonal()
    C = A.tocoo()
    keep = (C.row != C.col) & (blk[C.row] == blk[C.col]) & (np.abs(C.data) >= theta * np.sqrt(d[C.row] * d[C.col]))
    return sp.csr_matrix((np.ones(keep.sum()), (C.row[keep], C.col[keep])), shape=(n, n))


def _cases():
    out = []
    h = pscgen.poisson_hierarchy(7, 6, 5, max_levels=2)
    out.append(("poisson", h.levels[0].A.to_scipy(), [0, h.levels[0].n]))
    out.append(("poisson_l1", h.levels[1].A.to_scipy(), [0, h.levels[1].n]))
    h = pscgen.poisson_hierarchy(8, 6, 4, (2, 1, 1), max_levels=1)
    out.append(("poisson_2blocks", h.levels[0].A.to_scipy(), list(h.levels[0].row_start)))
    h = pscgen.poisson_hierarchy(8, problem="jump", cube=2, max_levels=1)
    out.append(("jump", h.levels[0].A.to_scipy(), [0, h.levels[0].n]))
    A = random_spd_mixed(60, 0.06, 3)
    out.append(("mixed_sign", A, [0, 30, 60]))
    return out


@pytest.mark.parametrize("name,A,rs", _cases(), ids=lambda c: c if isinstance(c, str) else "")
@pytest.mark.parametrize("theta", [0.01, 0.25])
def test_vmb_aggregation_rules(name, A, rs, theta):
    agg, root, nc = oracle.vmb_aggregate(A, theta, rs)
    n = A.shape[0]
    S = _strong(A, theta, rs)
    D = shortest_path(S, unweighted=True)
    roots = np.flatnonzero(root)
    # roots: pairwise more than two strong edges apart (no root is aggregated by another)
    sub = D[np.ix_(roots, roots)]
    assert np.all(sub[~np.eye(len(roots), dtype=bool)] >= 3)
    # greedy in increasing index (phase 1 visit order, R26): every non-root has a root
    # of smaller index within two strong edges -- with independence this is unique
    for v in np.flatnonzero(~root):
        near = roots[(D[v, roots] <= 2) & (roots < v)]
        assert len(near) > 0, v
    # ids: roots numbered in increasing index; a root and its strong neighbours share it
    assert nc == len(roots) and np.array_equal(agg[roots], np.arange(nc))
    assert agg.min() >= 0 and agg.max() == nc - 1  # disjoint and covering
    phase1 = np.zeros(n, bool)
    for r in roots:
        nb = S[r].indices
        assert np.all(agg[nb] == agg[r])
        phase1[nb] = True
        phase1[r] = True
    # phase 2 (R18): the strongest strong neighbour's phase-1 aggregate, ties
    # to the lowest id; strength |a_ij| / sqrt(a_ii a_jj)
    Ad = sp.csr_matrix(A)
    d = Ad.diagonal()
    for v in np.flatnonzero(~phase1):
        nb = [j for j in S[v].indices if phase1[j]]
        assert nb, v  # never phase 3
        st = np.array([abs(Ad[v, j]) / np.sqrt(d[v] * d[j]) for j in nb])
        best = [agg[j] for j, s in zip(nb, st) if s == st.max()]
        assert agg[v] == min(best)
    # decoupled: an aggregate never spans two row blocks
    blk = np.searchsorted(np.asarray(rs), np.arange(n), side="right") - 1
    for a in range(nc):
        assert len(np.unique(blk[agg == a])) == 1


def test_vmb_spec_examples():
    # diagonal matrix -> n singletons; path of 3 nodes, theta 0.25 -> {0,1,2};
    # two disconnected strongly coupled pairs -> 2 aggregates
    agg, root, nc = oracle.vmb_aggregate(sp.diags([1.0, 2.0, 3.0], format="csr"), 0.25)
    assert nc == 3 and np.array_equal(agg, [0, 1, 2])
    agg, root, nc = oracle.vmb_aggregate(tridiag(3), 0.25)
    assert nc == 1 and np.array_equal(agg, [0, 0, 0]) and np.array_equal(root, [True, False, False])
    pairs = sp.block_diag([tridiag(2), tridiag(2)], format="csr")
    agg, root, nc = oracle.vmb_aggregate(pairs, 0.25)
    assert nc == 2 and np.array_equal(agg, [0, 0, 1, 1])
    # theta = 0.6 on tridiag(-1,2,-1): |-1| < 0.6 * 2, no strong couplings
    agg, root, nc = oracle.vmb_aggregate(tridiag(5), 0.6)
    assert nc == 5


def test_omega_closed_forms():
    # tridiag(-1,2,-1) n = 2: ||D^-1 A||_inf = (2+1)/2 = 1.5
    assert oracle.omega(tridiag(2)) == 1.0 / golden("inf_norm_Dinv_A_tridiag_n2")
    assert oracle.omega(sp.diags([2.0, 5.0, 7.0], format="csr")) == 1.0  # D^-1 A = I
    # 7-point (6, -1) with an interior row: (6 + 6) / 6 = 2 -> omega = 1/2 ("~ 1/rho")
    A = pscgen.poisson_hierarchy(5, max_levels=1).levels[0].A.to_scipy()
    assert oracle.omega(A) == 0.5


def test_smoothed_prolongator_spec_examples():
    # A = I -> omega = 1, P = 0;  tridiag n = 2 with P^ = [1; 1] -> omega = 2/3, P = [2/3; 2/3]
    I3 = sp.eye(3, format="csr")
    P = oracle.smoothed_prolongator(I3, np.array([0, 1, 2]), 3, oracle.omega(I3))
    assert P.shape == (3, 3) and not P.toarray().any()
    A = tridiag(2)
    om = oracle.omega(A)
    assert om == 2.0 / 3.0
    P = oracle.smoothed_prolongator(A, np.array([0, 0]), 1, om)
    np.testing.assert_allclose(P.toarray(), [[2.0 / 3.0], [2.0 / 3.0]], rtol=1e-15)
    # Galerkin of [[2,-1],[-1,2]] with P = [1; 1] -> [2]
    P1 = sp.csr_matrix(np.ones((2, 1)))
    Ac = oracle.galerkin(oracle.transpose(P1), A, P1)
    assert np.array_equal(Ac.toarray(), golden("galerkin_2x2_p_ones"))


@pytest.mark.parametrize("name,A,rs", _cases(), ids=lambda c: c if isinstance(c, str) else "")
def test_prolongator_closed_forms(name, A, rs):
    A = sp.csr_matrix(A)
    agg, root, nc = oracle.vmb_aggregate(A, 0.01, rs)
    n = A.shape[0]
    # omega = 0 reduces to the tentative prolongator of Eq. (3), w = 1: one 1 per row, at agg(i)
    P0 = oracle.smoothed_prolongator(A, agg, nc, 0.0).toarray()
    Phat = np.zeros((n, nc))
    Phat[np.arange(n), agg] = 1.0
    assert np.array_equal(P0, Phat)
    om = oracle.omega(A)
    P = oracle.smoothed_prolongator(A, agg, nc, om)
    # P^ 1_c = 1, so P 1_c = (I - omega D^-1 A) 1
    d = A.diagonal()
    np.testing.assert_allclose(P @ np.ones(nc), 1.0 - om * (A @ np.ones(n)) / d, rtol=0, atol=1e-14)
    # P = P^ - omega D^-1 A P^ entry by entry (sparse library products as the steps)
    ref = Phat - om * (sp.diags(1.0 / d) @ A @ sp.csr_matrix(Phat)).toarray()
    np.testing.assert_allclose(P.toarray(), ref, rtol=0, atol=1e-14)
    # sparsity: an entry (i, J) only where row i of A reaches aggregate J
    reach = (abs(A) @ sp.csr_matrix(Phat)).toarray() != 0
    assert np.all(reach[P.toarray() != 0])
    # R = P^T exactly
    R = oracle.transpose(P)
    assert (R != P.T).nnz == 0 and np.all(np.diff(R.indptr) >= 0)


@pytest.mark.parametrize("name,A,rs", _cases()[:4], ids=lambda c: c if isinstance(c, str) else "")
def test_galerkin_bilinear_identity_symmetry_spd(name, A, rs):
    A = sp.csr_matrix(A)
    agg, root, nc = oracle.vmb_aggregate(A, 0.01, rs)
    P = oracle.smoothed_prolongator(A, agg, nc, oracle.omega(A))
    R = oracle.transpose(P)
    Ac = oracle.galerkin(R, A, P)
    rng = np.random.default_rng(4)
    for _ in range(3):
        x, y = rng.standard_normal(nc), rng.standard_normal(nc)
        lhs = x @ (Ac @ y)
        rhs = (P @ x) @ (A @ (P @ y))
        assert abs(lhs - rhs) <= 1e-12 * abs(P @ x).max() * abs(A).sum(axis=1).max() * abs(P @ y).max() * A.shape[0]
    np.testing.assert_allclose(Ac.toarray(), (P.T @ A @ P).toarray(), rtol=0, atol=1e-12 * abs(Ac).max())
    np.testing.assert_allclose(Ac.toarray(), Ac.toarray().T, rtol=0, atol=1e-13 * abs(Ac).max())
    assert np.linalg.eigvalsh(Ac.toarray()).min() > 0


def test_setup_hierarchy_vs_paper_fig3_and_generator():
    """Whole set-up on 64^3 Poisson: operator complexity near Fig. 3's VBM values
    (1.575 at 1 GPU; loose: +-0.03 -- the paper's matrix is 200^3 and its
    coarse-size target differs), A_{l+1} symmetric; the hierarchy equals the input
    generator's (an independent implementation of the same rules, pscgen) level by level."""
    g = 64
    hp = pscgen.poisson_hierarchy(g)
    H = oracle.amg_setup(hp.levels[0].A.to_scipy())
    assert abs(H.operator_complexity() - golden("vbm_operator_complexity_1gpu")) <= 0.03
    assert [L.n for L in H.levels] == [L.n for L in hp.levels]
    for l in range(H.nlevels):
        Ao, Ap = H.levels[l].A, hp.levels[l].A.to_scipy()
        assert (Ao != Ao.T).nnz == 0 or abs(Ao - Ao.T).max() <= 1e-13 * abs(Ao).max()
        assert abs(Ao - Ap).max() <= 1e-12 * abs(Ap).max()


@pytest.mark.slow
def test_setup_hierarchy_paper_fig2_iterations_loose():
    """P:380 (Fig. 2): VBM needs 18 iterations to 1e-6 at 1 GPU; with the oracle's own
    set-up at 128^3 (PCG, 30 coarse sweeps): within +-4."""
    g = 128
    A = pscgen.poisson_hierarchy(g, max_levels=1).levels[0].A.to_scipy()
    H = oracle.amg_setup(A)
    b = pscgen.rhs_poisson((g, g, g), 0, H.levels[0].n)
    x, it, st, hist = oracle.pcg(H, b, tol=1e-6, maxit=100)
    assert st == 0 and abs(it - golden("vbm_iterations_1gpu_tol1e-6")) <= 4
