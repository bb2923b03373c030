"""Pins of the oracle's AINV smoother (oracle/psc_oracle.c
or_ainv and the AINV branch of the V-cycle, reading R27): A^-1 ~ Z D^-1 Z^T
from an incomplete A-biconjugation, applied as x += Z D^-1 Z^T (b - A x).

Pinned against SPEC.md's worked examples, the exactness limit (drop 0:
Z D^-1 Z^T = A^-1; Z^T A Z = D), triangular structure, block-Jacobi
decoupling, the dense error-propagation form of Eq. (2) with G = I - Z D^-1 Z^T A,
symmetry of the resulting V-cycle, and an A-norm contraction.
"""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

import oracle
import pscgen
from _util import random_spd, random_spd_mixed, tridiag


def test_ainv_spec_examples():
    # diagonal A -> Z = I, D = diag(A), exact inverse
    A = sp.diags([2.0, 5.0, 0.5], format="csr")
    Z, p = oracle.ainv(A, 0.3)
    assert np.array_equal(Z.toarray(), np.eye(3)) and np.array_equal(p, [2.0, 5.0, 0.5])
    # [[2,-1],[-1,2]], drop 0 -> Z D^-1 Z^T = A^-1 = (1/3)[[2,1],[1,2]]
    Z, p = oracle.ainv(tridiag(2), 0.0)
    M = Z.toarray() @ np.diag(1.0 / p) @ Z.toarray().T
    np.testing.assert_allclose(M, np.array([[2.0, 1.0], [1.0, 2.0]]) / 3.0, rtol=0, atol=1e-12)
    # drop = inf -> Z = I, application = scaling by 1/pivots (= 1/a_ii)
    Z, p = oracle.ainv(tridiag(5), np.inf)
    assert np.array_equal(Z.toarray(), np.eye(5)) and np.array_equal(p, 2.0 * np.ones(5))


@pytest.mark.parametrize("seed", range(4))
def test_ainv_exactness_limit_and_conjugacy(seed):
    """drop 0 on SPD n <= 20: Z D^-1 Z^T = A^-1 (bound 1e-8) and Z^T A Z = D;
    Z unit upper triangular."""
    A = (random_spd(18, 0.25, seed) if seed % 2 else random_spd_mixed(18, 0.2, seed)).toarray()
    Z, p = oracle.ainv(sp.csr_matrix(A), 0.0)
    Zd = Z.toarray()
    assert np.array_equal(np.diag(Zd), np.ones(18)) and not np.tril(Zd, -1).any()
    np.testing.assert_allclose(Zd @ np.diag(1.0 / p) @ Zd.T, np.linalg.inv(A), rtol=0,
                               atol=1e-8 * np.abs(np.linalg.inv(A)).max())
    C = Zd.T @ A @ Zd
    np.testing.assert_allclose(C, np.diag(p), rtol=0, atol=1e-12 * np.abs(A).max() * 18)


def test_ainv_block_jacobi_decoupled():
    """Distributed form ('approximates the inversion of diagonal blocks'):
    with two row blocks, Z has no entry coupling the blocks and equals the AINV of
    each diagonal block."""
    A = random_spd(24, 0.3, 5)
    Z, p = oracle.ainv(A, 0.05, [0, 10, 24])
    Zd = Z.toarray()
    assert not Zd[:10, 10:].any() and not Zd[10:, :10].any()
    for a, b in ((0, 10), (10, 24)):
        Zb, pb = oracle.ainv(A[a:b, a:b], 0.05)
        np.testing.assert_array_equal(Zd[a:b, a:b], Zb.toarray())
        np.testing.assert_array_equal(p[a:b], pb)


def _block_ainv_dense(A, drop, rs):
    """Z D^-1 Z^T assembled from independent dense-block factors (block-Jacobi AINV)."""
    Ad = A.to_scipy().tocsr()
    n = Ad.shape[0]
    M = np.zeros((n, n))
    for a, b in zip(rs[:-1], rs[1:]):
        Zb, pb = oracle.ainv(Ad[a:b, a:b], drop)
        Zb = Zb.toarray()
        M[a:b, a:b] = Zb @ np.diag(1.0 / pb) @ Zb.T
    return M


def _dense_ainv_B(h, drop, pre, post, blocks=None):
    """B_0 of Eq. (2) with M_l^-1 = Z D^-1 Z^T (dense composition; coarsest: 30 l1 sweeps);
    blocks[l]: row starts of level l's AINV blocks (None: whole level)."""
    L = h.nlevels

    def Bl(l):
        A = h.levels[l].A.to_scipy().toarray()
        n = A.shape[0]
        if l == L - 1:
            m = np.abs(A).sum(axis=1)
            G = np.eye(n) - A / m[:, None]
            return (np.eye(n) - np.linalg.matrix_power(G, 30)) @ np.linalg.inv(A)
        rs = blocks[l] if blocks is not None and blocks[l] is not None else [0, n]
        Minv = _block_ainv_dense(h.levels[l].A, drop, rs)
        G = np.eye(n) - Minv @ A
        P = h.levels[l].P.to_scipy().toarray()
        R = h.levels[l].R.to_scipy().toarray()
        E = np.linalg.matrix_power(G, post) @ (np.eye(n) - P @ Bl(l + 1) @ R @ A) @ np.linalg.matrix_power(G, pre)
        return (np.eye(n) - E) @ np.linalg.inv(A)

    return Bl(0)


@pytest.mark.parametrize("drop,pre,post", [(0.1, 1, 1), (0.05, 2, 2), (0.2, 1, 2)])
def test_vcycle_with_ainv_equals_dense_eq2(drop, pre, post):
    h = pscgen.poisson_hierarchy(6, 5, 4, max_levels=3, coarse_target=4)
    n = h.levels[0].n
    B = _dense_ainv_B(h, drop, pre, post)
    for seed in (1, 2):
        r = pscgen.rhs_random(seed, 0, n)
        z = oracle.vcycle(h, r, pre=pre, post=post, smoother="ainv", ainv_drop=drop)
        np.testing.assert_allclose(z, B @ r, rtol=0, atol=1e-11 * np.abs(B @ r).max())
    if pre == post:  # symmetric smoother (M^-T = M^-1) and equal counts: B symmetric
        np.testing.assert_allclose(B, B.T, rtol=0, atol=1e-10 * np.abs(B).max())


def test_ainv_smoother_contracts_and_pcg_solves():
    h = pscgen.poisson_hierarchy(6, coarse_target=20)
    A = h.levels[0].A.to_scipy().toarray()
    Z, p = oracle.ainv(h.levels[0].A, 0.1)
    Zd = Z.toarray()
    G = np.eye(A.shape[0]) - Zd @ np.diag(1.0 / p) @ Zd.T @ A
    Lc = np.linalg.cholesky(A)
    # ||G||_A = ||L^T G L^-T||_2 < 1: the AINV smoother is A-convergent here
    assert np.linalg.norm(Lc.T @ G @ np.linalg.inv(Lc.T), 2) < 1.0
    b = pscgen.rhs_random(4, 0, A.shape[0])
    x, it, st, hist = oracle.pcg(h, b, tol=1e-12, maxit=200, pre=1, post=1, smoother="ainv", ainv_drop=0.1)
    assert st == 0
    xc = sla.cho_solve(sla.cho_factor(A), b)
    assert np.linalg.norm(x - xc) / np.linalg.norm(xc) < 1e-10


def test_vcycle_with_block_jacobi_ainv():
    """Per-level AINV blocks (the distributed form): the V-cycle equals the
    dense Eq. (2) composition with block-diagonal M_l^-1 built from independent block
    factors, differs from the whole-matrix smoother, and one block = the default."""
    h = pscgen.poisson_hierarchy(6, 5, 4, max_levels=3, coarse_target=4)
    n0, n1 = h.levels[0].n, h.levels[1].n
    blocks = [np.array([0, 37, 80, n0]), np.array([0, n1 // 2, n1]), None]
    B = _dense_ainv_B(h, 0.1, 1, 1, blocks)
    r = pscgen.rhs_random(3, 0, n0)
    z = oracle.vcycle(h, r, pre=1, post=1, smoother="ainv", ainv_drop=0.1, ainv_blocks=blocks)
    np.testing.assert_allclose(z, B @ r, rtol=0, atol=1e-11 * np.abs(B @ r).max())
    zw = oracle.vcycle(h, r, pre=1, post=1, smoother="ainv", ainv_drop=0.1)
    assert np.abs(z - zw).max() > 1e-6 * np.abs(zw).max()
    z1 = oracle.vcycle(h, r, pre=1, post=1, smoother="ainv", ainv_drop=0.1,
                       ainv_blocks=[np.array([0, n0]), None, None])
    np.testing.assert_array_equal(z1, zw)
